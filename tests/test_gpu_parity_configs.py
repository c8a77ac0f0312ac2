"""GPU parity at the BASELINE configurations not covered elsewhere (VERDICT r1
"close the untested configs"):

* the layout pre-pass (geometry.py:257-380) on the configs[1] mesh, bit-exact
  against a fixture written by the reference itself (make_golden.py cfg2areas);
* configs[3]: the dense layout uniform_layout(mesh, 8) (10.8M texels, an
  accumulator far beyond L2), mul, c = 40;
* the full configs[1] job: 2000 frames, mul + images_iid, float32 accumulator;
* the furnished room (occlusion, 3-8 covering records per pixel): accumulators
  and labels, not just ids.

Bars: counts exact; float32 accumulators within 1e-5 of the
float64 oracle relative to max(|ref|, 1e-3) (log space for mul);
labels identical wherever the reference's top-2 margin is above 1e-5.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2111_11103_b200 import Mesh, MeshAnnotation, build_texel_layout, compute_worst_case_areas, uniform_layout
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics, pack_camera
from paper_2111_11103_b200.synth import make_furnished_room, make_room, random_room_trajectory, scannet_intrinsics, \
    softmax_maps

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
W, H = 640, 480


def _room():
    v, t = make_room((6.0, 5.0, 3.0), 158)
    return Mesh.from_arrays(v, t)


def _oracle_fold(mesh, layout, frames, probs_host, agg, nthreads=0):
    cams = np.stack([pack_camera(f) for f in frames])
    return O.fuse_frames_c(mesh.vertices, mesh.triangles, layout.steps, layout.origins, layout.offsets,
                           layout.total_texels, cams, W, H, probs_host, agg, "images_iid", nthreads=nthreads)


def _check(acc_got, cnt_got, lab_got, acc_ref, cnt_ref, agg):
    np.testing.assert_array_equal(cnt_got, cnt_ref)
    seen = cnt_ref > 0
    err = np.abs(acc_got[seen] - acc_ref[seen]) / np.maximum(np.abs(acc_ref[seen]), 1e-3)
    assert err.max() < 1e-5, err.max()
    rows, unobs = O.finalize(acc_ref, cnt_ref, agg)
    ref_lab = O.texel_argmax(rows, unobs)
    srt = np.sort(acc_ref, axis=1)
    if agg == "mul":
        decided = (srt[:, -1] - srt[:, -2]) >= 1e-5 * np.maximum(np.abs(acc_ref).max(axis=1), 1e-30)
    else:
        top2 = np.sort(rows.astype(np.float64), axis=1)[:, -2:]
        decided = (top2[:, 1] - top2[:, 0]) >= 1e-5
    decided |= unobs
    np.testing.assert_array_equal(lab_got[decided], ref_lab[decided])
    assert decided[seen].mean() > 0.99


def test_layout_prepass_cfg2_golden():
    """compute_worst_case_areas on the GPU == the reference's, bit for bit; the gamma 0.2 / 1.0
    layouts (ceil(gamma * sqrt(a)) boundaries) follow."""
    z = np.load(os.path.join(GOLD, "cfg2_areas.npz"))
    mesh = _room()
    intr = Intrinsics(577.87, 577.87, 319.5, 239.5, W, H)
    frames = [CameraFrame(k, intr, c[:9].reshape(3, 3), c[9:12]) for k, c in enumerate(z["cams"])]
    areas = compute_worst_case_areas(mesh, frames)
    np.testing.assert_array_equal(areas, z["areas"])
    for gamma in (0.2, 1.0):
        lay = build_texel_layout(mesh, areas, gamma)
        np.testing.assert_array_equal(lay.steps, z["steps_%g" % gamma])
        np.testing.assert_array_equal(lay.origins, z["origins_%g" % gamma])
        assert lay.total_texels == int(z["total_%g" % gamma])
    assert (z["steps_1"] > 1).sum() > 1000  # the fine layout has real subdivision


def test_cfg4_dense_layout_mul_vs_oracle():
    """configs[3]: uniform_layout(mesh, 8) -> 36 texels per triangle, 10,784,448 texels, a 1.73 GB
    float32 accumulator; 4 frames of c = 40 softmax maps, mul + images_iid."""
    mesh = _room()
    layout = uniform_layout(mesh, 8)
    assert layout.total_texels == 10784448
    frames = random_room_trajectory(4, scannet_intrinsics(), seed=31)
    probs = softmax_maps(4, H, W, 40, seed=3)
    ann = MeshAnnotation(mesh, layout, num_classes=40, aggregator="mul", accum_dtype="float32", max_batch=4)
    ann.add_batch(probs, frames)
    tex = ann.texture
    cnt_dev = tex._counts
    seen_dev = torch.nonzero(cnt_dev > 0).squeeze(1)
    acc_seen = tex._accum[seen_dev, :40].double().cpu().numpy()
    labels = ann.labels()
    lab_seen = labels[seen_dev].cpu().numpy()
    assert bool((labels[cnt_dev == 0] == -1).all())
    acc_ref, cnt_ref = _oracle_fold(mesh, layout, frames, list(probs.cpu().numpy()), "mul", nthreads=1)
    idx = seen_dev.cpu().numpy()
    assert np.array_equal(np.nonzero(cnt_ref)[0], idx)
    _check(acc_seen, cnt_dev[seen_dev].cpu().numpy(), lab_seen, acc_ref[idx], cnt_ref[idx], "mul")


def test_cfg2_full_job_2000_frames_vs_oracle():
    """configs[1] end to end: the bench workload (2000 frames cycling an 8-map pool, mul + images_iid,
    float32 accumulator, batches of 256) against the float64 C oracle over the same frames."""
    mesh = _room()
    layout = uniform_layout(mesh, 1)
    frames = random_room_trajectory(2000, scannet_intrinsics(), seed=1000)
    pool = softmax_maps(8, H, W, 40, seed=0)
    ann = MeshAnnotation(mesh, layout, num_classes=40, aggregator="mul", accum_dtype="float32", max_batch=256)
    ann.add_batch([pool[i % 8] for i in range(2000)], frames)
    acc = ann.texture.accum
    cnt = ann.texture.counts
    labels = ann.labels(host=True)
    host_pool = list(pool.cpu().numpy())
    acc_ref, cnt_ref = _oracle_fold(mesh, layout, frames, [host_pool[i % 8] for i in range(2000)], "mul")
    _check(acc, cnt, labels, acc_ref, cnt_ref, "mul")
    assert (cnt_ref > 0).mean() > 0.9 and cnt_ref.max() > 1000  # many adds per texel: the A3 regime


@pytest.mark.parametrize("agg", ["mul", "sum"])
def test_furnished_room_accumulators_and_labels(agg):
    """cfg2 + furniture (3-8 covering records per pixel over the boxes): the depth test decides
    which texel each pixel feeds; accumulators, counts and labels vs the oracle."""
    v, t = make_furnished_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(12, scannet_intrinsics(), seed=21)
    probs = softmax_maps(12, H, W, 40, seed=9)
    ann = MeshAnnotation(mesh, layout, num_classes=40, aggregator=agg, accum_dtype="float32", max_batch=5)
    ann.add_batch(probs, frames)
    acc_ref, cnt_ref = _oracle_fold(mesh, layout, frames, list(probs.cpu().numpy()), agg)
    assert (cnt_ref[layout.offsets[299568]:] > 0).sum() > 1000  # furniture texels observed
    _check(ann.texture.accum, ann.texture.counts, ann.labels(host=True), acc_ref, cnt_ref, agg)

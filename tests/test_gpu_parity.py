"""GPU parity: the CUDA path against the reference goldens and the CPU oracle.

Bars: triangle / texel ids bit-exact (depth, u, v too);
counts exact; float64 accumulators within 1e-12 relative (atomic order),
float32 accumulators within 1e-5 relative (log space for mul); labels
identical except where the reference's top-2 margin is below 1e-5.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_2111_11103_b200 import (
    MeshAnnotation, Mesh, TexelLayout, accumulate_frame, build_texel_layout, compute_pixel_weights,
    compute_worst_case_areas, finalize, init_texture, rasterize, render_labels, texel_argmax, uniform_layout)
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics, pack_camera
from paper_2111_11103_b200.rasterizer import IdImage
from paper_2111_11103_b200.synth import (NoiseModel, corrupt, make_room, random_room_trajectory,
                                         scannet_intrinsics)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _frame(cam, W, H, fid=0):
    return CameraFrame(fid, Intrinsics(cam[12], cam[13], cam[14], cam[15], W, H), cam[:9].reshape(3, 3), cam[9:12])


@pytest.fixture(scope="module")
def cfg1():
    z = np.load(os.path.join(GOLD, "cfg1.npz"))
    d = {k: z[k] for k in z.files}
    mesh = Mesh(d["verts"], d["tris"])
    layout = TexelLayout(d["steps"], d["origins"], d["offsets"], int(d["total_texels"]))
    W, H = (int(x) for x in d["wh"])
    frames = [_frame(c, W, H, i) for i, c in enumerate(d["cams"])]
    c = int(d["num_classes"])
    model = NoiseModel("flip", epsilon=0.3, q=0.8, seed=1)
    probs = [corrupt(d["gt"][f].astype(np.int32), model, c, f) for f in range(len(frames))]
    return d, mesh, layout, frames, probs


def test_raster_golden_cases_bitexact():
    z = np.load(os.path.join(GOLD, "raster_cases.npz"))
    for name in [str(n) for n in z["names"]]:
        mesh = Mesh(z[name + "/verts"], z[name + "/tris"])
        steps = z[name + "/steps"]
        layout = TexelLayout(steps, z[name + "/origins"], z[name + "/offsets"],
                             int(((steps.astype(np.int64) ** 2 + steps) // 2).sum()))
        W, H = (int(x) for x in z[name + "/wh"])
        for f, cam in enumerate(z[name + "/cams"]):
            ids = rasterize(mesh, layout, _frame(cam, W, H))
            np.testing.assert_array_equal(ids.triangle, z[name + "/tri"][f], err_msg=name)
            np.testing.assert_array_equal(ids.texel, z[name + "/texel"][f], err_msg=name)
            np.testing.assert_array_equal(ids.depth, z[name + "/depth"][f], err_msg=name)
            cov = ids.triangle >= 0
            np.testing.assert_array_equal(ids.u[cov], z[name + "/u"][f][cov], err_msg=name)
            np.testing.assert_array_equal(ids.v[cov], z[name + "/v"][f][cov], err_msg=name)


def test_raster_cfg1_all_frames_bitexact(cfg1):
    d, mesh, layout, frames, _ = cfg1
    for f, fr in enumerate(frames):
        ids = rasterize(mesh, layout, fr)
        np.testing.assert_array_equal(ids.triangle, d["tri"][f])
        np.testing.assert_array_equal(ids.texel, d["texel"][f])


def test_raster_cfg2_full_frame_bitexact():
    z = np.load(os.path.join(GOLD, "cfg2_frame.npz"))
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    ids = rasterize(mesh, layout, _frame(z["cam"], 640, 480))
    np.testing.assert_array_equal(ids.triangle, z["tri"])
    np.testing.assert_array_equal(ids.texel, z["texel"])
    assert float(ids.depth[ids.covered].sum()) == float(z["depth_sum"])


def test_raster_cfg2_batched_random_cameras_vs_oracle():
    """Full BASELINE size, batched launch (B=6), fine layout (steps=3): rows bit-exact."""
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 3)
    frames = random_room_trajectory(6, scannet_intrinsics(), seed=11)
    ann = MeshAnnotation(mesh, layout, num_classes=4, max_batch=6)
    cams = ann.scene.cams_tensor(frames)
    rows = torch.empty((6, 640 * 480), dtype=torch.int32, device=ann.device)
    ann.scene.rasterize(cams, 640, 480, rows)
    rows = rows.cpu().numpy()
    for k, fr in enumerate(frames):
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 640, 480,
                          want_uv=False)
        np.testing.assert_array_equal(rows[k], O.pixel_rows(layout.offsets, ref["triangle"], ref["texel"]).ravel())


def test_raster_overflow_fallback_exact():
    """A pair capacity far too small forces every tile through the exact slow path."""
    from paper_2111_11103_b200 import _native as N

    v, t = make_room((6.0, 5.0, 3.0), 24)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(2, Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96), seed=5)
    ann = MeshAnnotation(mesh, layout, num_classes=4, max_batch=2)
    sc = ann.scene
    cams = sc.cams_tensor(frames)
    nbytes = N.load().tfb_raster_workspace_bytes(mesh.num_vertices, mesh.num_triangles, 128, 96, 2, 16)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=ann.device)
    rows = torch.empty((2, 128 * 96), dtype=torch.int32, device=ann.device)
    N.call("tfb_rasterize", sc.sref, N.ptr(cams), 2, 128, 96, N.ptr(ws), nbytes, 16, N.ptr(rows), None, None, None,
           None, None, None, N.stream_handle())
    rows = rows.cpu().numpy()
    for k, fr in enumerate(frames):
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 128, 96,
                          want_uv=False)
        np.testing.assert_array_equal(rows[k], O.pixel_rows(layout.offsets, ref["triangle"], ref["texel"]).ravel())


def test_worst_case_areas_and_layout_cfg1(cfg1):
    d, mesh, _, frames, _ = cfg1
    areas = compute_worst_case_areas(mesh, frames)
    np.testing.assert_array_equal(areas, d["areas"])
    layout = build_texel_layout(mesh, areas, 0.2)
    np.testing.assert_array_equal(layout.steps, d["steps"])
    np.testing.assert_array_equal(layout.offsets, d["offsets"])
    np.testing.assert_array_equal(layout.origins, d["origins"])


def _margin_ok(rows_ref, unobs_ref, labels_ref, labels, agg, accum_ref):
    top2 = np.sort(rows_ref.astype(np.float64), axis=1)[:, -2:]
    if agg == "mul":
        scale = np.abs(accum_ref).max(axis=1)
        gap = (np.sort(accum_ref, axis=1)[:, -1] - np.sort(accum_ref, axis=1)[:, -2])
        decided = gap >= 1e-5 * np.maximum(scale, 1e-30)
    else:
        decided = (top2[:, 1] - top2[:, 0]) >= 1e-5
    decided &= top2[:, 1] != top2[:, 0]
    decided |= unobs_ref
    np.testing.assert_array_equal(labels[decided], labels_ref[decided])
    return decided


@pytest.mark.parametrize("agg", ["sum", "mul", "maxsum"])
@pytest.mark.parametrize("wm", ["images_iid", "pixels_iid"])
def test_fusion_cfg1_float64_library_api(cfg1, agg, wm):
    d, mesh, layout, frames, probs = cfg1
    key = "%s_%s" % (agg, wm)
    tex = init_texture(layout, int(d["num_classes"]), agg, accum_dtype="float64")
    for fr, p in zip(frames, probs):
        ids = rasterize(mesh, layout, fr)
        accumulate_frame(tex, ids, p, compute_pixel_weights(ids, wm))
    np.testing.assert_array_equal(tex.counts, d[key + "/counts"])
    ref = d[key + "/accum"]
    np.testing.assert_allclose(tex.accum, ref, rtol=1e-12, atol=1e-12)
    finalize(tex)
    np.testing.assert_array_equal(tex.unobserved, d[key + "/unobserved"])
    np.testing.assert_allclose(tex.rows, d[key + "/rows"], atol=1e-6)
    labels = texel_argmax(tex)
    _margin_ok(d[key + "/rows"], d[key + "/unobserved"], d[key + "/labels"], labels, agg, ref)
    if key + "/rendered" in d:
        for f, (fr, p) in enumerate(zip(frames, probs)):
            ids = rasterize(mesh, layout, fr)
            out = render_labels(d[key + "/labels"], layout, ids, fallback=p.argmax(axis=2).astype(np.int32))
            np.testing.assert_array_equal(out, d[key + "/rendered"][f])


@pytest.mark.parametrize("agg", ["sum", "mul", "maxsum"])
def test_fusion_cfg1_float32_batched(cfg1, agg):
    d, mesh, layout, frames, probs = cfg1
    key = "%s_images_iid" % agg
    ann = MeshAnnotation(mesh, layout, num_classes=int(d["num_classes"]), aggregator=agg,
                         weight_mode="images_iid", accum_dtype="float32", max_batch=7)
    ann.add_batch(torch.as_tensor(np.stack(probs)).cuda(), frames)
    np.testing.assert_array_equal(ann.texture.counts, d[key + "/counts"])
    ref = d[key + "/accum"]
    got = ann.texture.accum
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)
    assert err.max() < 1e-5, err.max()
    labels = ann.labels(host=True)
    _margin_ok(d[key + "/rows"], d[key + "/unobserved"], d[key + "/labels"], labels, agg, ref)


def test_fusion_cfg2_float32_mul_vs_oracle():
    """BASELINE size: 6 frames, c=40 softmax maps, mul + images_iid, vs the float64 oracle."""
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    frames = random_room_trajectory(6, scannet_intrinsics(), seed=2)
    g = torch.Generator(device="cuda").manual_seed(7)
    probs = torch.softmax(torch.randn((6, 480, 640, 40), generator=g, device="cuda") * 2, dim=-1)
    ann = MeshAnnotation(mesh, layout, num_classes=40, aggregator="mul", weight_mode="images_iid", max_batch=4)
    fb = torch.empty((6, 480 * 640), dtype=torch.int32, device="cuda")
    ann.add_batch(probs, frames, fallback_out=fb)
    acc = np.zeros((layout.total_texels, 40))
    cnt = np.zeros(layout.total_texels, np.int64)
    ph = probs.cpu().numpy()
    for k, fr in enumerate(frames):
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 640, 480,
                          want_uv=False)
        w = O.compute_pixel_weights(ref["triangle"], ref["texel"], "images_iid")
        O.accumulate_frame(acc, cnt, layout.offsets, ref["triangle"], ref["texel"], ph[k], w, "mul")
        np.testing.assert_array_equal(fb[k].cpu().numpy(), ph[k].argmax(axis=2).ravel())
    np.testing.assert_array_equal(ann.texture.counts, cnt)
    got = ann.texture.accum
    seen = cnt > 0
    err = np.abs(got[seen] - acc[seen]) / np.maximum(np.abs(acc[seen]), 1e-3)
    assert err.max() < 1e-5, err.max()
    rows, unobs = O.finalize(acc, cnt, "mul")
    _margin_ok(rows, unobs, O.texel_argmax(rows, unobs), ann.labels(host=True), "mul", acc)


def test_render_batched_matches_oracle(cfg1):
    d, mesh, layout, frames, probs = cfg1
    key = "sum_images_iid"
    ann = MeshAnnotation(mesh, layout, num_classes=int(d["num_classes"]), aggregator="sum",
                         accum_dtype="float64", max_batch=8)
    ann.add_batch(probs, frames)
    labels = ann.labels(host=True)
    imgs = ann.render(frames, host=True)
    for f in range(len(frames)):
        ref = O.render_labels(labels, layout.offsets, d["tri"][f], d["texel"][f])
        np.testing.assert_array_equal(imgs[f], ref)
    _margin_ok(d[key + "/rows"], d[key + "/unobserved"], d[key + "/labels"], labels, "sum", d[key + "/accum"])


def test_host_ids_rows_and_weights():
    mesh = Mesh.from_arrays(np.array([[0, 0, 1], [1, 0, 1], [0, 1, 1.0]]), np.array([[0, 1, 2]]))
    layout = uniform_layout(mesh, 3)
    ids = IdImage(0, 4, 1, triangle=np.array([[0, 0, -1, 0]]), texel=np.array([[1, 1, 0, 5]]))
    w = compute_pixel_weights(ids, "images_iid")
    np.testing.assert_allclose(np.asarray(w), [[0.5, 0.5, 0.0, 1.0]])
    tex = init_texture(layout, 2, "sum")
    accumulate_frame(tex, ids, np.full((1, 4, 2), 0.5, np.float32), w)
    assert tex.counts.tolist() == [0, 2, 0, 0, 0, 1]


def test_raster_dense_tiles_big_path_exact():
    """Tiles holding more records than a k_raster CTA stages (> 128 per 16x8
    tile): k_raster_big's list mode, with heavy overlap (many candidates per
    pixel, near-coplanar stacks) — ids, depth, u, v bit-exact vs the oracle."""
    rng = np.random.default_rng(21)
    m = 1500
    # small triangles packed into a 40x24-pixel window 2 m in front of the camera,
    # at depths 1.9..2.1 (many overlaps, several exactly coplanar groups)
    centers = np.column_stack([rng.uniform(-0.2, 0.2, m), rng.uniform(-0.12, 0.12, m),
                               np.round(rng.uniform(1.9, 2.1, m), 2)])
    offs = rng.uniform(-0.03, 0.03, size=(m, 3, 3))
    offs[:, :, 2] *= 0.1
    verts = (centers[:, None, :] + offs).reshape(-1, 3)
    tris = np.arange(3 * m, dtype=np.int32).reshape(m, 3)
    mesh = Mesh.from_arrays(verts, tris)
    layout = uniform_layout(mesh, 3)
    W, H = 96, 64
    fr = CameraFrame(0, Intrinsics(200.0, 200.0, 47.5, 31.5, W, H), np.eye(3), np.zeros(3))
    ids = rasterize(mesh, layout, fr)
    ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), W, H)
    np.testing.assert_array_equal(ids.triangle, ref["triangle"])
    np.testing.assert_array_equal(ids.texel, ref["texel"])
    np.testing.assert_array_equal(ids.depth, ref["depth"])
    cov = ids.triangle >= 0
    np.testing.assert_array_equal(ids.u[cov], ref["u"][cov])
    np.testing.assert_array_equal(ids.v[cov], ref["v"][cov])
    assert cov.mean() > 0.1  # the 40x24-pixel window is covered


@pytest.mark.parametrize("m", [60, 400, 700])
def test_raster_tile_tiers_exact(m):
    """Record densities that put the window's 16x8 tiles in each rasterizer tier:
    <= 64 records (k_raster<64>), 64 < n <= 128 (the 128-thread tier kernel
    walking its list) and beyond (k_raster_big), with overlapping stacks -- ids,
    depth, u, v bit-exact vs the oracle."""
    rng = np.random.default_rng(100 + m)
    centers = np.column_stack([rng.uniform(-0.2, 0.2, m), rng.uniform(-0.12, 0.12, m),
                               np.round(rng.uniform(1.9, 2.1, m), 2)])
    offs = rng.uniform(-0.04, 0.04, size=(m, 3, 3))
    offs[:, :, 2] *= 0.1
    verts = (centers[:, None, :] + offs).reshape(-1, 3)
    mesh = Mesh.from_arrays(verts, np.arange(3 * m, dtype=np.int32).reshape(m, 3))
    layout = uniform_layout(mesh, 2)
    W, H = 96, 64
    fr = CameraFrame(0, Intrinsics(200.0, 200.0, 47.5, 31.5, W, H), np.eye(3), np.zeros(3))
    ids = rasterize(mesh, layout, fr)
    ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), W, H)
    for key, plane in (("triangle", ids.triangle), ("texel", ids.texel), ("depth", ids.depth)):
        np.testing.assert_array_equal(plane, ref[key], err_msg=key)
    cov = ids.triangle >= 0
    np.testing.assert_array_equal(ids.u[cov], ref["u"][cov])
    np.testing.assert_array_equal(ids.v[cov], ref["v"][cov])
    assert cov.mean() > 0.02


def _raster_rows_hits(mesh, layout, frames, W, H, clusters, monkeypatch):
    from paper_2111_11103_b200.device import DeviceScene

    monkeypatch.setenv("TFB_NO_CLUSTERS", "0" if clusters else "1")
    sc = DeviceScene(mesh, layout)
    assert (sc.clusters is not None) == clusters
    cams = sc.cams_tensor(frames)
    B = len(frames)
    rows = torch.empty((B, W * H), dtype=torch.int32, device=sc.device)
    hits = torch.zeros((B, layout.total_texels), dtype=torch.int32, device=sc.device)
    tri = torch.empty((B, W * H), dtype=torch.int32, device=sc.device)
    tex = torch.empty((B, W * H), dtype=torch.int32, device=sc.device)
    sc.rasterize(cams, W, H, rows, hits, tri, tex)
    return rows.cpu().numpy(), hits.cpu().numpy(), tri.cpu().numpy(), tex.cpu().numpy()


def test_raster_cluster_cull_identical(monkeypatch):
    """The cluster cull (tfb_scene clusters) drops only clusters that produce no
    pixel: ids and hit counts equal the per-triangle cull's, including cameras
    grazing walls, in corners and looking along a wall (clusters straddling the
    near plane and the image edges)."""
    from paper_2111_11103_b200.synth import look_at

    v, t = make_room((6.0, 5.0, 3.0), 40)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    intr = Intrinsics(300.0, 300.0, 159.5, 119.5, 320, 240)
    frames = list(random_room_trajectory(24, intr, seed=3))
    special = [((2.999, 0.0, 0.0), (3.0, 1.0, 0.0)), ((2.9999, 2.4999, 1.4999), (0.0, 0.0, 0.0)),
               ((0.0, 0.0, 1.49995), (1.0, 0.0, 1.49995)), ((-2.99, -2.49, -1.49), (-2.99, 2.0, -1.49)),
               ((0.0, 2.49999, 0.0), (0.0, 0.0, 0.0)), ((1.0, 1.0, 0.0), (1.0, 1.0, -1.0))]
    for k, (eye, target) in enumerate(special):
        R, tr = look_at(np.array(eye), np.array(target))
        frames.append(CameraFrame(100 + k, intr, R, tr))
    a = _raster_rows_hits(mesh, layout, frames, 320, 240, True, monkeypatch)
    b = _raster_rows_hits(mesh, layout, frames, 320, 240, False, monkeypatch)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    for k in (0, len(frames) - 3, len(frames) - 1):  # and both equal the oracle
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(frames[k]), 320,
                          240, want_uv=False)
        np.testing.assert_array_equal(a[2][k], ref["triangle"].ravel())


def test_raster_cluster_cull_sphere_outside(monkeypatch):
    """A convex object seen from outside (back faces and a silhouette), clusters vs none."""
    from paper_2111_11103_b200.synth import look_at, make_icosphere

    mesh = make_icosphere(1.0, 4)
    layout = uniform_layout(mesh, 1)
    intr = Intrinsics(200.0, 200.0, 79.5, 59.5, 160, 120)
    rng = np.random.default_rng(7)
    frames = []
    for k in range(16):
        d = rng.normal(size=3)
        eye = d / np.linalg.norm(d) * rng.uniform(1.05, 4.0)
        R, tr = look_at(eye, rng.normal(size=3) * 0.5)
        frames.append(CameraFrame(k, intr, R, tr))
    a = _raster_rows_hits(mesh, layout, frames, 160, 120, True, monkeypatch)
    b = _raster_rows_hits(mesh, layout, frames, 160, 120, False, monkeypatch)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)



def test_raster_furnished_room_vs_oracle():
    """cfg2 with furniture (SURVEY §7 hard part 9): occlusion, so pixels with
    several covering records and the depth test; rows bit-exact at 640x480 for
    a batch, and one frame's tri / texel / depth / u / v through rasterize()."""
    from paper_2111_11103_b200.synth import make_furnished_room

    v, t = make_furnished_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(4, scannet_intrinsics(), seed=21)
    ann = MeshAnnotation(mesh, layout, num_classes=4, max_batch=4)
    cams = ann.scene.cams_tensor(frames)
    rows = torch.empty((4, 640 * 480), dtype=torch.int32, device=ann.device)
    ann.scene.rasterize(cams, 640, 480, rows)
    rows = rows.cpu().numpy()
    box_pixels = 0
    for k, fr in enumerate(frames):
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 640, 480,
                          want_uv=(k == 0))
        np.testing.assert_array_equal(rows[k], O.pixel_rows(layout.offsets, ref["triangle"], ref["texel"]).ravel())
        box_pixels += int((ref["triangle"] >= 299568).sum())
        if k == 0:
            ids = rasterize(mesh, layout, fr)
            np.testing.assert_array_equal(ids.triangle, ref["triangle"])
            np.testing.assert_array_equal(ids.texel, ref["texel"])
            np.testing.assert_array_equal(ids.depth, ref["depth"])
            np.testing.assert_array_equal(ids.u, ref["u"])
            np.testing.assert_array_equal(ids.v, ref["v"])
    assert box_pixels > 1000  # the furniture is in view and occludes the walls


def test_raster_large_triangles_few_survivors():
    """Triangles spanning every tile with only 1-3 survivors in a frame (a
    partial warp in k_setup bins a wide record cooperatively): ids equal the
    oracle's."""
    v = np.array([[-10, -10, 5], [10, -10, 5], [0, 10, 5]], dtype=np.float64)
    for ntri in (1, 2, 3, 40):
        vs = np.concatenate([v + [0.01 * k, 0.02 * k, k * 0.1] for k in range(ntri)])
        t = np.arange(3 * ntri, dtype=np.int32).reshape(ntri, 3)
        mesh = Mesh.from_arrays(vs, t)
        layout = uniform_layout(mesh, 2)
        fr = CameraFrame(0, Intrinsics(32.0, 32.0, 31.5, 31.5, 64, 64), np.eye(3), np.zeros(3))
        ids = rasterize(mesh, layout, fr)
        ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 64, 64,
                          want_uv=False)
        np.testing.assert_array_equal(ids.triangle, ref["triangle"])
        np.testing.assert_array_equal(ids.texel, ref["texel"])
        assert (ids.triangle >= 0).mean() > 0.5


@pytest.mark.parametrize("layers", [2, 3, 4, 5, 8, 9, 14])
def test_raster_stacked_layers_vs_oracle(layers):
    """`layers` overlapping triangles in front of each other (shuffled order,
    some nearly coplanar), so pixels hold 2..14 covering records: the 2-slot,
    4-input-network, kept-slot selection and full-scan fold paths; ids, depth,
    u, v bit-exact with the oracle."""
    rng = np.random.default_rng(layers)
    base = np.array([[-1.0, -1.0, 0.0], [1.2, -0.9, 0.0], [0.1, 1.1, 0.0]])
    vs, ts = [], []
    for k in rng.permutation(layers):
        z = 3.0 + 0.05 * k + (1e-10 if k % 3 == 0 else 0.0)
        tri = base * (1.0 + 0.03 * k) + [0.02 * k, -0.01 * k, z]
        vs.append(tri)
        ts.append(np.arange(3) + 3 * len(ts))
    mesh = Mesh.from_arrays(np.concatenate(vs), np.array(ts, dtype=np.int32))
    layout = uniform_layout(mesh, 3)
    fr = CameraFrame(0, Intrinsics(60.0, 60.0, 39.5, 29.5, 80, 60), np.eye(3), np.zeros(3))
    ids = rasterize(mesh, layout, fr)
    ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 80, 60)
    for key, plane in (("triangle", ids.triangle), ("texel", ids.texel), ("depth", ids.depth)):
        np.testing.assert_array_equal(plane, ref[key], err_msg=key)
    cov = ids.triangle >= 0
    np.testing.assert_array_equal(ids.u[cov], ref["u"][cov])
    np.testing.assert_array_equal(ids.v[cov], ref["v"][cov])


def test_raster_cfg5_scale_frame_vs_oracle():
    """BASELINE cfg5 scale: the 5M-triangle room at 1920x1080 (ids of one
    frame bit-exact with the C oracle; clusters, large bins, every kernel at
    full size)."""
    v, t = make_room((6.0, 5.0, 3.0), 646)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    intr = Intrinsics(1728.0, 1728.0, 959.5, 539.5, 1920, 1080)
    fr = random_room_trajectory(1, intr, seed=17)[0]
    ann = MeshAnnotation(mesh, layout, num_classes=4, max_batch=1)
    cams = ann.scene.cams_tensor([fr])
    rows = torch.empty((1, 1920 * 1080), dtype=torch.int32, device=ann.device)
    ann.scene.rasterize(cams, 1920, 1080, rows)
    ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), 1920, 1080,
                      want_uv=False)
    np.testing.assert_array_equal(rows[0].cpu().numpy(), O.pixel_rows(layout.offsets, ref["triangle"],
                                                                       ref["texel"]).ravel())


def test_raster_odd_image_sizes_vs_oracle():
    """Image sizes that are not multiples of the 16x8 tile (partial tiles on
    both edges), with clusters and tile bins, rows bit-exact."""
    v, t = make_room((6.0, 5.0, 3.0), 30)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    for W, H in ((97, 61), (17, 9), (1, 1), (33, 200)):
        intr = Intrinsics(0.9 * W, 0.9 * W, (W - 1) / 2.0, (H - 1) / 2.0, W, H)
        frames = random_room_trajectory(3, intr, seed=W + H)
        ann = MeshAnnotation(mesh, layout, num_classes=4, max_batch=3)
        cams = ann.scene.cams_tensor(frames)
        rows = torch.empty((3, W * H), dtype=torch.int32, device=ann.device)
        ann.scene.rasterize(cams, W, H, rows)
        rows = rows.cpu().numpy()
        for k, fr in enumerate(frames):
            ref = O.rasterize(mesh.vertices, mesh.triangles, layout.steps, layout.origins, pack_camera(fr), W, H,
                              want_uv=False)
            np.testing.assert_array_equal(rows[k], O.pixel_rows(layout.offsets, ref["triangle"],
                                                                ref["texel"]).ravel(), err_msg="%dx%d" % (W, H))


@pytest.mark.parametrize("agg", ["sum", "maxsum", "mul"])
@pytest.mark.parametrize("accum_dtype", ["float32", "float64"])
def test_accumulate_frame_explicit_random_weights_vs_oracle(agg, accum_dtype):
    """accumulate_frame with a caller-provided per-pixel weight array that
    varies inside texel runs (the scatter-add's per-pixel weight path), and
    probabilities hitting the clip bounds, vs the float64 oracle."""
    v, t = make_room((6.0, 5.0, 3.0), 12)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    intr = Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96)
    frames = random_room_trajectory(3, intr, seed=8)
    rng = np.random.default_rng(3)
    tex = init_texture(layout, 5, agg, accum_dtype=accum_dtype)
    acc = np.zeros((layout.total_texels, 5))
    cnt = np.zeros(layout.total_texels, np.int64)
    for fr in frames:
        ids = rasterize(mesh, layout, fr)
        p = rng.dirichlet(np.ones(5), size=(96, 128)).astype(np.float32)
        p[::7, ::5, 1] = 0.0
        p[::11, ::3, 2] = 1.0
        w = rng.uniform(0.0, 3.0, size=(96, 128))
        accumulate_frame(tex, ids, p, w)
        O.accumulate_frame(acc, cnt, layout.offsets, ids.triangle, ids.texel, p, w, agg)
    got = tex.accum
    np.testing.assert_array_equal(tex.counts, cnt)
    tol = 1e-5 if accum_dtype == "float32" else 1e-12
    scale = np.abs(acc).max(axis=1, keepdims=True) + 1e-30
    assert (np.abs(got - acc) / scale).max() < tol

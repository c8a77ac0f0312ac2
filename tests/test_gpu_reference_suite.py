"""The reference's own test expectations, run through the GPU drop-in API.

Ports of /root/reference/pkg/tests/test_fusion.py, test_rasterizer.py,
test_renderback.py (render/fusion parts), test_acceptance.py criteria 2, 3, 4,
5, 7, 8, 10 and bindings/tests/test_session.py — same inputs, same closed-form
oracles, same tolerances (1e-6 rows need the float64 accumulator, the
library API's default).
"""

import math
import threading

import numpy as np
import pytest

import paper_2111_11103_b200 as tf
from paper_2111_11103_b200 import (AGGREGATORS, UNKNOWN, CapacityError, DataError, Mesh, accumulate_frame,
                                   build_texel_layout, compute_pixel_weights, compute_worst_case_areas, finalize,
                                   init_texture, rasterize, render_labels, texel_argmax, texel_count,
                                   uniform_layout)
from paper_2111_11103_b200.fusion import MUL_CLAMP
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics
from paper_2111_11103_b200.rasterizer import NONE, IdImage, pixel_world_points
from paper_2111_11103_b200.synth import (NoiseModel, corrupt, make_cube, make_icosphere, make_orbit_trajectory)

pytestmark = pytest.mark.gpu


# ----------------------------------------------------------------- helpers (tests/helpers.py)
def frontal_frame(width=64, height=64, fx=None, frame_id=0):
    fx = float(width) if fx is None else fx
    intr = Intrinsics(fx=fx, fy=fx, cx=width / 2.0, cy=height / 2.0, width=width, height=height)
    return CameraFrame(frame_id=frame_id, intrinsics=intr, rotation=np.eye(3), translation=np.zeros(3))


def strip_mesh(n, z=0.0):
    verts, tris = [], []
    for k in range(n):
        x = 2.0 * k
        verts += [(x, 0.0, z), (x + 1.0, 0.0, z), (x, 1.0, z)]
        tris.append((3 * k, 3 * k + 1, 3 * k + 2))
    return Mesh.from_arrays(np.array(verts, dtype=np.float64), np.array(tris, dtype=np.int32))


def square_mesh(half=0.5, z=2.0):
    verts = np.array([[-half, -half, z], [half, -half, z], [half, half, z], [-half, half, z]])
    return Mesh.from_arrays(verts, np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int32))


def handmade_ids(triangle, texel, width=None, height=1, frame_id=0):
    tri = np.asarray(triangle, dtype=np.int32)
    tex = np.asarray(texel, dtype=np.int32)
    if width is None:
        width = tri.size // height
    return IdImage(frame_id, width, height, triangle=tri.reshape(height, width), texel=tex.reshape(height, width))


def _texture(num_classes=2, triangles=1, aggregator="sum"):
    mesh = strip_mesh(triangles)
    return init_texture(build_texel_layout(mesh, np.zeros(triangles), 0.0), num_classes, aggregator)


def _probs(rows):
    arr = np.asarray(rows, dtype=np.float32)
    return arr.reshape(1, len(rows), -1)


def _unit(n):
    return np.ones((1, n), dtype=np.float64)


# ----------------------------------------------------------------- test_fusion.py
def test_reference_vectors():
    for agg, p, want in (("sum", [[0.6, 0.4], [0.2, 0.8]], [0.4, 0.6]),
                         ("mul", [[0.6, 0.4], [0.6, 0.4]], [9 / 13, 4 / 13]),
                         ("maxsum", [[0.6, 0.4], [0.45, 0.55]], [0.6 / 1.15, 0.55 / 1.15])):
        tex = _texture(aggregator=agg)
        accumulate_frame(tex, handmade_ids([0, 0], [0, 0]), _probs(p), _unit(2))
        finalize(tex)
        np.testing.assert_allclose(tex.rows[0], want, atol=1e-6)


def test_maxsum_keeps_all_tied_maxima():
    tex = _texture(num_classes=3, aggregator="maxsum")
    accumulate_frame(tex, handmade_ids([0], [0]), _probs([[0.4, 0.4, 0.2]]), _unit(1))
    finalize(tex)
    np.testing.assert_allclose(tex.rows[0], [0.5, 0.5, 0.0], atol=1e-7)


def test_sum_finalize_normalizes_accumulator():
    tex = _texture(aggregator="sum")
    accumulate_frame(tex, handmade_ids([0], [0]), _probs([[0.25, 0.75]]), np.full((1, 1), 8.0))
    np.testing.assert_allclose(tex.accum[0], [2.0, 6.0], atol=1e-12)
    finalize(tex)
    np.testing.assert_allclose(tex.rows[0], [0.25, 0.75], atol=1e-12)


def test_mul_finalize_survives_extreme_logs():
    tex = _texture(aggregator="mul")
    tex.accum[0] = [-700.0, -710.0]
    tex.counts[0] = 1
    finalize(tex)
    row = tex.rows[0]
    assert np.isfinite(row).all()
    np.testing.assert_allclose(row.sum(), 1.0, atol=1e-6)
    np.testing.assert_allclose(row[0], 1.0 / (1.0 + np.exp(-10.0)), atol=1e-6)


def test_unobserved_zero_weight_and_empty():
    tex = _texture(num_classes=4, triangles=3)
    accumulate_frame(tex, handmade_ids([1], [0]), _probs([[0.7, 0.1, 0.1, 0.1]]), _unit(1))
    finalize(tex)
    assert tex.unobserved.tolist() == [True, False, True]
    np.testing.assert_allclose(tex.rows[0], 0.25)
    assert tex.counts.tolist() == [0, 1, 0]
    tex = _texture(num_classes=2)
    accumulate_frame(tex, handmade_ids([0], [0]), _probs([[0.9, 0.1]]), np.zeros((1, 1)))
    finalize(tex)
    assert bool(tex.unobserved[0])
    np.testing.assert_allclose(tex.rows[0], 0.5)
    tex = _texture(num_classes=3, triangles=2)
    finalize(tex)
    assert tex.unobserved.all()
    np.testing.assert_allclose(tex.rows, 1.0 / 3.0)


def test_guards_and_shape_checks():
    tex = _texture()
    finalize(tex)
    with pytest.raises(RuntimeError):
        finalize(tex)
    with pytest.raises(RuntimeError):
        accumulate_frame(tex, handmade_ids([0], [0]), _probs([[0.5, 0.5]]), _unit(1))
    with pytest.raises(RuntimeError):
        texel_argmax(_texture())
    tex = _texture(num_classes=3)
    ids = handmade_ids([0, 0], [0, 0])
    with pytest.raises(DataError):
        accumulate_frame(tex, ids, _probs([[0.5, 0.5], [0.5, 0.5]]), _unit(2))
    with pytest.raises(DataError):
        accumulate_frame(tex, ids, _probs([[0.3, 0.3, 0.4], [0.3, 0.3, 0.4]]), np.ones((2, 2)))


def test_texel_argmax_examples():
    mesh = strip_mesh(3)
    tex = init_texture(build_texel_layout(mesh, np.zeros(3), 0.0), 3, "sum")
    accumulate_frame(tex, handmade_ids([0, 1], [0, 0]), _probs([[0.1, 0.7, 0.2], [0.5, 0.5, 0.0]]), _unit(2))
    finalize(tex)
    labels = texel_argmax(tex)
    assert labels.tolist() == [1, 0, UNKNOWN]


def test_pixel_weight_modes():
    ids = handmade_ids([0, 0, 0, 0], [0, 0, 0, 0])
    np.testing.assert_allclose(compute_pixel_weights(ids, "pixels_iid"), 1.0)
    np.testing.assert_allclose(compute_pixel_weights(ids, "images_iid"), 0.25)
    np.testing.assert_allclose(compute_pixel_weights(ids, "blend", 0.5), 0.5 * 1.0 + 0.5 * 0.25)
    w = compute_pixel_weights(handmade_ids([0, -1], [0, 0]), "images_iid")
    assert w[0, 0] == 1.0 and w[0, 1] == 0.0
    rng = np.random.default_rng(2)
    tri = rng.integers(-1, 3, size=30)
    tex = rng.integers(0, 2, size=30)
    ids = handmade_ids(tri, np.where(tri >= 0, tex, 0), height=5, width=6)
    np.testing.assert_array_equal(compute_pixel_weights(ids, "blend", 0.0), compute_pixel_weights(ids, "pixels_iid"))
    np.testing.assert_array_equal(compute_pixel_weights(ids, "blend", 1.0), compute_pixel_weights(ids, "images_iid"))
    rng = np.random.default_rng(9)
    tri = rng.integers(-1, 5, size=400)
    texel = rng.integers(0, 3, size=400)
    ids = handmade_ids(tri, np.where(tri >= 0, texel, 0), height=20, width=20)
    w = np.asarray(compute_pixel_weights(ids, "images_iid"))
    cov = tri.reshape(20, 20) >= 0
    key = ids.triangle[cov].astype(np.int64) * 3 + ids.texel[cov]
    sums = np.bincount(key, weights=w[cov])
    np.testing.assert_allclose(sums[np.bincount(key) > 0], 1.0, atol=1e-6)


def test_mul_argmax_invariant_to_scaling_and_replication_and_order():
    rows = [[0.5, 0.3, 0.2], [0.2, 0.5, 0.3], [0.6, 0.2, 0.2]]
    out = []
    for scale in (1.0, 0.07):
        tex = _texture(num_classes=3, aggregator="mul")
        accumulate_frame(tex, handmade_ids([0, 0, 0], [0, 0, 0]),
                         (np.asarray(rows, np.float32) * scale).reshape(1, 3, 3), _unit(3))
        finalize(tex)
        out.append(int(np.argmax(tex.rows[0])))
    assert out[0] == out[1]
    rng = np.random.default_rng(4)
    for agg in AGGREGATORS:
        reps = rng.integers(1, 5, size=6)
        p = rng.random((6, 3)).astype(np.float32) + 0.05
        p /= p.sum(axis=1, keepdims=True)
        tw = _texture(num_classes=3, aggregator=agg)
        accumulate_frame(tw, handmade_ids([0] * 6, [0] * 6), p.reshape(1, 6, 3), reps.astype(np.float64).reshape(1, 6))
        finalize(tw)
        tr = _texture(num_classes=3, aggregator=agg)
        flat = np.repeat(p, reps, axis=0)
        accumulate_frame(tr, handmade_ids([0] * len(flat), [0] * len(flat)), flat.reshape(1, len(flat), 3),
                         _unit(len(flat)))
        finalize(tr)
        np.testing.assert_allclose(tw.rows[0], tr.rows[0], atol=1e-6)
    rng = np.random.default_rng(8)
    p = rng.random((10, 4)).astype(np.float32) + 0.01
    p /= p.sum(axis=1, keepdims=True)
    w = rng.uniform(0.1, 2.0, size=10)
    for agg in AGGREGATORS:
        ref = None
        for seed in range(3):
            tex = _texture(num_classes=4, aggregator=agg)
            for k in np.random.default_rng(seed).permutation(10):
                accumulate_frame(tex, handmade_ids([0], [0], frame_id=int(k)), p[k].reshape(1, 1, 4),
                                 np.full((1, 1), w[k]))
            finalize(tex)
            ref = tex.rows[0].copy() if ref is None else ref
            np.testing.assert_allclose(tex.rows[0], ref, atol=1e-6)


# ----------------------------------------------------------------- test_acceptance.py c2, c3, c8
def _oracle_rows(agg, p, w):
    p64 = p.astype(np.float64)
    if agg == "sum":
        r = (w[:, None] * p64).sum(axis=0)
    elif agg == "maxsum":
        keep = p64 == p64.max(axis=1, keepdims=True)
        r = (w[:, None] * np.where(keep, p64, 0.0)).sum(axis=0)
    else:
        r = np.prod(np.clip(p64, MUL_CLAMP, 1.0) ** w[:, None], axis=0)
    return r / r.sum()


def _fuse_rows(agg, p, w):
    tex = init_texture(build_texel_layout(strip_mesh(1), np.zeros(1), 0.0), p.shape[1], agg)
    n = len(p)
    accumulate_frame(tex, handmade_ids([0] * n, [0] * n), p.reshape(1, n, -1), w.reshape(1, n))
    finalize(tex)
    return tex.rows[0].astype(np.float64)


def test_criterion_02_aggregator_oracle_suite():
    rng = np.random.default_rng(2026)
    worst = 0.0
    for case in range(1000):
        n = int(rng.integers(1, 11))
        c = int(rng.integers(2, 6))
        p = (rng.random((n, c)) + 1e-3).astype(np.float32)
        p /= p.sum(axis=1, keepdims=True)
        w = rng.uniform(0.05, 3.0, size=n)
        agg = AGGREGATORS[case % 3]
        worst = max(worst, np.abs(_fuse_rows(agg, p, w) - _oracle_rows(agg, p, w)).max())
    assert worst < 1e-6, worst


def test_criterion_03_permutation_invariance():
    rng = np.random.default_rng(33)
    mesh = strip_mesh(3)
    layout = build_texel_layout(mesh, np.array([0.0, 9.0, 100.0]), 0.4)
    worst = 0.0
    for case in range(100):
        n = int(rng.integers(2, 31))
        c = int(rng.integers(2, 5))
        agg = AGGREGATORS[case % 3]
        tri = rng.integers(0, 3, size=n)
        tex_ids = np.array([rng.integers(0, texel_count(int(layout.steps[t]))) for t in tri])
        p = (rng.random((n, c)) + 1e-3).astype(np.float32)
        p /= p.sum(axis=1, keepdims=True)
        w = rng.uniform(0.1, 2.0, size=n)
        rows = []
        for perm_seed in (0, 1):
            order = np.random.default_rng((case, perm_seed)).permutation(n)
            tex = init_texture(layout, c, agg)
            cuts = sorted(rng.integers(0, n, size=2))
            for lo, hi in zip([0] + cuts, cuts + [n]):
                if lo == hi:
                    continue
                sel = order[lo:hi]
                accumulate_frame(tex, handmade_ids(tri[sel], tex_ids[sel], frame_id=lo),
                                 p[sel].reshape(1, len(sel), c), w[sel].reshape(1, len(sel)))
            finalize(tex)
            rows.append(tex.rows.astype(np.float64))
        worst = max(worst, np.abs(rows[0] - rows[1]).max())
    assert worst < 1e-6, worst


def test_criterion_08_weight_replication():
    rng = np.random.default_rng(88)
    worst = 0.0
    for case in range(200):
        agg = AGGREGATORS[case % 3]
        n = int(rng.integers(1, 9))
        c = int(rng.integers(2, 6))
        reps = rng.integers(1, 5, size=n)
        p = (rng.random((n, c)) + 1e-3).astype(np.float32)
        p /= p.sum(axis=1, keepdims=True)
        a = _fuse_rows(agg, p, reps.astype(np.float64))
        b = _fuse_rows(agg, np.repeat(p, reps, axis=0), np.ones(int(reps.sum())))
        worst = max(worst, float(np.abs(a - b).max()))
    assert worst < 1e-6, worst


# ----------------------------------------------------------------- test_rasterizer.py
def test_rasterizer_behaviour():
    mesh = Mesh.from_arrays(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int32))
    ids = rasterize(mesh, uniform_layout(mesh), frontal_frame())
    assert (ids.triangle == NONE).all() and np.isinf(ids.depth).all()
    near, far = square_mesh(0.4, 1.0), square_mesh(0.4, 2.0)
    mesh = Mesh.from_arrays(np.vstack([far.vertices, near.vertices]), np.vstack([far.triangles, near.triangles + 4]))
    ids = rasterize(mesh, uniform_layout(mesh), frontal_frame(64, 64, 64.0))
    cov = ids.covered
    assert cov.any() and (ids.triangle[cov] >= 2).all()
    np.testing.assert_allclose(ids.depth[cov], 1.0, atol=1e-9)
    one = square_mesh(0.4, 2.0)
    mesh = Mesh.from_arrays(np.vstack([one.vertices, one.vertices]), np.vstack([one.triangles, one.triangles + 4]))
    ids = rasterize(mesh, uniform_layout(mesh), frontal_frame(64, 64, 64.0))
    assert (ids.triangle[ids.covered] <= 1).all()
    mesh = square_mesh(0.45, 1.5)
    ids = rasterize(mesh, uniform_layout(mesh), frontal_frame(96, 96, 96.0))
    lo, hi = int(np.ceil(48 - 0.45 / 1.5 * 96)) + 1, int(np.floor(48 + 0.45 / 1.5 * 96)) - 1
    assert ids.covered[lo:hi, lo:hi].all()
    assert (np.bincount(ids.triangle[ids.covered], minlength=2) > 0).all()
    assert not rasterize(square_mesh(0.4, -2.0), uniform_layout(square_mesh(0.4, -2.0)), frontal_frame()).covered.any()


def test_rasterizer_invariants_on_cube_orbit():
    scene = make_cube()
    layout = uniform_layout(scene, steps=6)
    intr = frontal_frame(64, 48, 48.0).intrinsics
    for frame in make_orbit_trajectory((0, 0, 0), 3.0, 6, intr, tilt_deg=20.0):
        ids = rasterize(scene, layout, frame)
        cov = ids.covered
        assert cov.any() and (ids.depth[cov] > 0).all()
        u, v = ids.u[cov], ids.v[cov]
        assert (0.0 <= v).all() and (v <= u).all() and (u <= 1.0).all()
        assert (ids.texel[cov] < texel_count(layout.steps[ids.triangle[cov]])).all()
        assert np.isinf(ids.depth[~cov]).all()


def test_interior_uv_is_perspective_correct():
    frame = frontal_frame(64, 64, 64.0)
    screen = [(10.5, 10.5), (50.5, 12.5), (12.5, 52.5)]
    verts = [((px - 32.0) / 64.0 * z, (py - 32.0) / 64.0 * z, z) for (px, py), z in zip(screen, (1.0, 2.0, 3.0))]
    mesh = Mesh.from_arrays(np.array(verts), np.array([[0, 1, 2]]))
    layout = uniform_layout(mesh, 7)
    ids = rasterize(mesh, layout, frame)
    cov = ids.covered
    ys, xs = np.nonzero(cov)
    v0, v1, v2 = mesh.vertices[mesh.triangles[0]]
    n = np.cross(v1 - v0, v2 - v0)
    rays = np.stack([(xs + 0.5 - 32.0) / 64.0, (ys + 0.5 - 32.0) / 64.0, np.ones_like(xs, dtype=np.float64)], axis=1)
    t = (v0 @ n) / (rays @ n)
    hit = rays * t[:, None]
    area = np.linalg.norm(n)
    b0 = np.einsum("ij,ij->i", np.cross(v1 - hit, v2 - hit), n[None, :]) / area ** 2
    b1 = np.einsum("ij,ij->i", np.cross(v2 - hit, v0 - hit), n[None, :]) / area ** 2
    b = np.stack([b0, b1, 1.0 - b0 - b1])
    o = int(layout.origins[0])
    np.testing.assert_allclose(ids.u[cov], np.clip(1.0 - b[o], 0, 1), atol=1e-6)
    np.testing.assert_allclose(ids.v[cov], np.clip(b[(o + 2) % 3], 0, None), atol=1e-6)
    np.testing.assert_allclose(ids.depth[cov], t, rtol=1e-9)


def test_pixel_world_points_reproject():
    scene = make_cube()
    layout = uniform_layout(scene, steps=3)
    frame = make_orbit_trajectory((0, 0, 0), 3.0, 5, frontal_frame(64, 48, 48.0).intrinsics, tilt_deg=15.0)[2]
    ids = rasterize(scene, layout, frame)
    pts = pixel_world_points(scene, layout, ids)
    ys, xs = np.nonzero(ids.covered)
    cam = (frame.rotation @ pts.T).T + frame.translation
    np.testing.assert_allclose(cam[:, 0] / cam[:, 2] * frame.fx + frame.cx, xs + 0.5, atol=1e-6)
    np.testing.assert_allclose(cam[:, 2], ids.depth[ids.covered], rtol=1e-9)


# ----------------------------------------------------------------- c4: rasterizer vs ray cast
def _random_scene(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(5, 51))
    centers = np.stack([rng.uniform(-1.2, 1.2, m), rng.uniform(-1.2, 1.2, m), rng.uniform(1.5, 4.0, m)], axis=1)
    verts = (centers[:, None, :] + rng.normal(scale=0.45, size=(m, 3, 3))).reshape(-1, 3)
    verts[:, 2] = np.maximum(verts[:, 2], 0.3)
    return Mesh.from_arrays(verts, np.arange(3 * m).reshape(m, 3))


def _raycast(mesh, fx, cx, n):
    px, py = np.meshgrid(np.arange(n) + 0.5, np.arange(n) + 0.5)
    dirs = np.stack([(px - cx) / fx, (py - cx) / fx, np.ones_like(px)], axis=2)
    best_z = np.full((n, n), np.inf)
    best_t = np.full((n, n), -1, dtype=np.int32)
    V = mesh.vertices[mesh.triangles]
    for t in range(len(V)):
        v0, v1, v2 = V[t]
        nrm = np.cross(v1 - v0, v2 - v0)
        with np.errstate(divide="ignore", invalid="ignore"):
            z = (v0 @ nrm) / (dirs @ nrm)
        q = dirs * z[..., None]
        c0 = np.cross(v1 - v0, q - v0) @ nrm
        c1 = np.cross(v2 - v1, q - v1) @ nrm
        c2 = np.cross(v0 - v2, q - v2) @ nrm
        same = ((c0 >= 0) & (c1 >= 0) & (c2 >= 0)) | ((c0 <= 0) & (c1 <= 0) & (c2 <= 0))
        better = np.isfinite(z) & (z > 0) & same & (z < best_z - 1e-12)
        best_z[better] = z[better]
        best_t[better] = t
    return best_t, best_z


def test_criterion_04_rasterizer_vs_raycast():
    frame = frontal_frame(64, 64, 64.0)
    union = agree = 0
    worst = 0.0
    for seed in range(20):
        mesh = _random_scene(seed)
        ids = rasterize(mesh, uniform_layout(mesh), frame)
        ot, oz = _raycast(mesh, 64.0, 32.0, 64)
        u = ids.covered | (ot >= 0)
        a = ids.covered & (ot >= 0) & (ids.triangle == ot)
        union += int(u.sum())
        agree += int(a.sum())
        if a.any():
            worst = max(worst, float(np.abs(ids.depth[a] - oz[a]).max()))
    assert agree / union >= 0.99 and worst <= 1e-6


# ----------------------------------------------------------------- c5 / c7 / c10: end to end
def _accuracy(pred, ref, c):
    valid = (ref >= 0) & (ref < c)
    return int((pred[valid] == ref[valid]).sum()), int(valid.sum())


def _gt(mesh, frame, labels_fn=None, face_labels=None):
    ids = rasterize(mesh, uniform_layout(mesh), frame)
    out = np.full((ids.height, ids.width), UNKNOWN, dtype=np.int32)
    cov = ids.covered
    if face_labels is not None:
        out[cov] = face_labels[ids.triangle[cov]]
    else:
        out[cov] = labels_fn(pixel_world_points(mesh, uniform_layout(mesh), ids))
    return out


def _orbit_fusion(mesh, c, frames, model, gamma, agg, wmode, gt_fn, subset=None):
    used = list(range(len(frames))) if subset is None else list(subset)
    layout = build_texel_layout(mesh, compute_worst_case_areas(mesh, [frames[k] for k in used]), gamma)
    ids_all, gts, probs = [], [], []
    for fr in frames:
        ids_all.append(rasterize(mesh, layout, fr))
        g = gt_fn(fr)
        gts.append(g)
        probs.append(corrupt(g, model, c, fr.frame_id))
    tex = init_texture(layout, c, agg)
    for k in used:
        accumulate_frame(tex, ids_all[k], probs[k], compute_pixel_weights(ids_all[k], wmode))
    finalize(tex)
    labels = texel_argmax(tex)
    bc = bn = fc = fn = 0
    for ids, g, p in zip(ids_all, gts, probs):
        raw = p.argmax(axis=2).astype(np.int32)
        out = render_labels(labels, layout, ids, fallback=raw)
        a, b = _accuracy(raw, g, c)
        bc, bn = bc + a, bn + b
        a, b = _accuracy(out, g, c)
        fc, fn = fc + a, fn + b
    return bc / bn, fc / fn


def test_criterion_05_end_to_end_fusion_gain():
    cube = make_cube()
    face = np.repeat(np.arange(6), 2).astype(np.int32)
    intr = Intrinsics(fx=96, fy=96, cx=48, cy=36, width=96, height=72)
    frames = make_orbit_trajectory((0, 0, 0), 3.0, 30, intr)
    model = NoiseModel(kind="flip", epsilon=0.3, q=0.8, seed=20260816)
    base, fused = _orbit_fusion(cube, 6, frames, model, 0.2, "mul", "images_iid",
                                lambda fr: _gt(cube, fr, face_labels=face))
    assert abs(base - 0.70) <= 0.01 and fused >= 0.99, (base, fused)


def test_criterion_06_frame_fraction_monotonicity():
    # test_acceptance.py:273-293: mean fused accuracy over 5 noise seeds is
    # non-decreasing in the fraction of frames fused (0.5 pt slack) and
    # saturated by half of the frames
    from paper_2111_11103_b200.renderback import select_frames

    cube = make_cube()
    face = np.repeat(np.arange(6), 2).astype(np.int32)
    intr = Intrinsics(fx=64, fy=64, cx=32, cy=24, width=64, height=48)
    frames = make_orbit_trajectory((0, 0, 0), 3.0, 20, intr)
    fractions = (0.05, 0.1, 0.2, 0.5, 1.0)
    curves = []
    for seed in range(5):
        model = NoiseModel(kind="flip", epsilon=0.35, q=0.7, seed=100 + seed)
        curves.append([_orbit_fusion(cube, 6, frames, model, 0.2, "mul", "images_iid",
                                     lambda fr: _gt(cube, fr, face_labels=face),
                                     subset=select_frames(len(frames), frac))[1] for frac in fractions])
    mean = np.mean(curves, axis=0)
    assert (np.diff(mean) >= -0.005).all(), mean
    assert abs(mean[-1] - mean[-2]) <= 0.005, mean


def test_criterion_07_weighting_separation():
    verts = np.array([[-0.3, -0.3, 0.0], [0.4, -0.2, 0.0], [0.0, 0.45, 0.0]]) * 0.5
    mesh = Mesh.from_arrays(verts, np.array([[0, 1, 2]]))
    layout = build_texel_layout(mesh, np.zeros(1), 0.0)
    p_near = np.array([0.2, 0.8], dtype=np.float32)
    p_far = np.array([0.8, 0.2], dtype=np.float32)
    views = []
    near = frontal_frame(64, 64, 64.0, 0)
    near.translation = np.array([0.0, 0.0, 0.5])
    views.append((near, p_near))
    for k in range(9):
        far = frontal_frame(64, 64, 64.0, 1 + k)
        far.translation = np.array([0.0, 0.0, 5.0])
        views.append((far, p_far))
    res, counts = {}, {}
    for mode in ("pixels_iid", "images_iid"):
        tex = init_texture(layout, 2, "sum")
        px = []
        for frame, pv in views:
            ids = rasterize(mesh, layout, frame)
            px.append(int(ids.covered.sum()))
            accumulate_frame(tex, ids, np.broadcast_to(pv, (64, 64, 2)).copy(), compute_pixel_weights(ids, mode))
        finalize(tex)
        counts[mode] = px
        res[mode] = (tex.accum[0].copy(), int(np.argmax(tex.rows[0])))
    n_near, n_far = counts["pixels_iid"][0], sum(counts["pixels_iid"][1:])
    assert n_near > 10 * n_far
    ap, amp = res["pixels_iid"]
    ai, ami = res["images_iid"]
    assert np.abs(ap - (n_near * p_near.astype(np.float64) + n_far * p_far.astype(np.float64))).max() < 1e-6 * n_near
    assert np.abs(ai - (1.0 * p_near.astype(np.float64) + 9.0 * p_far.astype(np.float64))).max() < 1e-6
    assert amp == 1 and ami == 0


def _checker_labels(level, num_classes):
    period = 36.0 / (2 ** level)

    def labels(points):
        points = np.asarray(points, dtype=np.float64)
        r = np.linalg.norm(points, axis=1)
        r = np.where(r == 0.0, 1.0, r)
        theta = np.degrees(np.arccos(np.clip(points[:, 2] / r, -1.0, 1.0)))
        az = np.degrees(np.arctan2(points[:, 1], points[:, 0])) % 360.0
        cell = np.floor(theta / period).astype(np.int64) + np.floor(az / period).astype(np.int64)
        return (cell % num_classes).astype(np.int32)

    return labels


def test_criterion_10_gamma_sensitivity_frozen_goldens():
    # test_acceptance.py:404-424: frozen accuracies {0.0: 0.524529, 0.5: 0.784785} at 1e-6
    sphere = make_icosphere(1.0, 2)
    lab = _checker_labels(2, 2)
    intr = Intrinsics(fx=128, fy=128, cx=64, cy=48, width=128, height=96)
    frames = make_orbit_trajectory((0, 0, 0), 3.0, 16, intr, tilt_deg=20.0)
    model = NoiseModel(kind="flip", epsilon=0.3, q=0.8, seed=3)
    acc = {g: _orbit_fusion(sphere, 2, frames, model, g, "mul", "images_iid",
                            lambda fr: _gt(sphere, fr, labels_fn=lab))[1] for g in (0.0, 0.5)}
    assert acc[0.5] >= acc[0.0] + 0.01
    assert abs(acc[0.0] - 0.524529) < 1e-6, acc
    assert abs(acc[0.5] - 0.784785) < 1e-6, acc


# ----------------------------------------------------------------- test_renderback.py
def test_render_labels_fallback_and_checks():
    mesh = square_mesh(0.4, 2.0)
    layout = uniform_layout(mesh)
    ids = rasterize(mesh, layout, frontal_frame(32, 32, 32.0))
    out = render_labels(np.array([3, UNKNOWN], np.int32), layout, ids)
    cov = ids.covered
    assert (out[~cov] == UNKNOWN).all()
    assert set(np.unique(out[cov])) <= {3, UNKNOWN}
    fb = np.full((32, 32), 7, np.int32)
    out2 = render_labels(np.array([3, UNKNOWN], np.int32), layout, ids, fallback=fb)
    assert (out2[out == UNKNOWN] == 7).all() and (out2[out == 3] == 3).all()
    with pytest.raises(DataError):
        render_labels(np.array([1, 2, 3]), layout, ids)
    with pytest.raises(DataError):
        render_labels(np.array([1, 2]), layout, ids, fallback=np.zeros((3, 3), np.int32))


def test_single_frame_fusion_equals_per_triangle_mean():
    scene = make_cube()
    frame = frontal_frame(64, 48, 48.0)
    frame.translation = np.array([0.0, 0.0, 3.0])
    layout = build_texel_layout(scene, np.zeros(scene.num_triangles), 0.0)
    ids = rasterize(scene, layout, frame)
    rng = np.random.default_rng(12)
    probs = rng.random((48, 64, 4)).astype(np.float32) + 0.01
    probs /= probs.sum(axis=2, keepdims=True)
    tex = init_texture(layout, 4, "sum")
    accumulate_frame(tex, ids, probs, np.ones((48, 64)))
    finalize(tex)
    cov = ids.covered
    tris = ids.triangle[cov]
    for t in np.unique(tris):
        want = probs[cov][tris == t].astype(np.float64).mean(axis=0)
        np.testing.assert_allclose(tex.rows[t], want / want.sum(), atol=1e-6)
    assert (texel_argmax(tex)[np.unique(tris)] != UNKNOWN).all()


# ----------------------------------------------------------------- bindings/tests/test_session.py
@pytest.fixture(scope="module")
def scene_dir(tmp_path_factory):
    out = tmp_path_factory.mktemp("bindings")
    cube = make_cube()
    face = np.repeat(np.arange(6), 2).astype(np.int32)
    intr = Intrinsics(fx=64.0, fy=64.0, cx=32.0, cy=24.0, width=64, height=48)
    frames = make_orbit_trajectory((0.0, 0.0, 0.0), 3.0, 8, intr, tilt_deg=25.0)
    tf.save_ply(out / "mesh.ply", cube)
    tf.save_trajectory(out / "trajectory.txt", frames)
    mesh = tf.load_mesh(out / "mesh.ply")
    model = NoiseModel("flip", 0.3, 0.8, seed=23)
    probs = {f.frame_id: corrupt(_gt(mesh, f, face_labels=face), model, 6, f.frame_id) for f in frames}
    return out, probs


def _fresh(scene_dir, gamma=0.2):
    return tf.open_session(scene_dir[0] / "mesh.ply", scene_dir[0] / "trajectory.txt", gamma, "mul", "images_iid", 6)


def test_session_layout_and_counts(scene_dir):
    ses = _fresh(scene_dir, 0.0)
    assert ses.num_texels == 12 and ses.num_classes == 6 and not ses.finalized
    ses = _fresh(scene_dir)
    assert ses.num_texels > 12
    added = tf.add_frame(ses, 0, scene_dir[1][0])
    assert 0 < added <= 64 * 48
    assert tf.add_frame(ses, 0, scene_dir[1][0]) == added
    sloppy = np.asfortranarray(scene_dir[1][2].astype(np.float64))
    assert tf.add_frame(ses, 2, sloppy) == tf.add_frame(ses, 2, scene_dir[1][2])
    with pytest.raises(DataError, match="99"):
        tf.add_frame(ses, 99, scene_dir[1][0])
    with pytest.raises(DataError, match="shape"):
        tf.add_frame(ses, 0, scene_dir[1][0].transpose(1, 0, 2))
    with pytest.raises(ValueError, match="outside"):
        tf.open_session(scene_dir[0] / "mesh.ply", scene_dir[0] / "trajectory.txt", 0.2, "mul", "blend:2.0", 6)


def test_session_rejects_concurrent_add_frame(scene_dir, monkeypatch):
    import paper_2111_11103_b200.session as S

    ses = _fresh(scene_dir)
    inside, release = threading.Event(), threading.Event()
    real = S.rasterize

    def stalled(*a, **k):
        inside.set()
        assert release.wait(10.0)
        return real(*a, **k)

    monkeypatch.setattr(S, "rasterize", stalled)
    worker = threading.Thread(target=S.add_frame, args=(ses, 0, scene_dir[1][0]))
    worker.start()
    try:
        assert inside.wait(10.0)
        with pytest.raises(RuntimeError, match="add_frame"):
            S.add_frame(ses, 1, scene_dir[1][1])
    finally:
        release.set()
        worker.join(10.0)
    assert int(ses.texture.counts.sum()) > 0


def test_session_finalize_and_render(scene_dir):
    ses = _fresh(scene_dir)
    tf.add_frame(ses, 0, scene_dir[1][0])
    with pytest.raises(DataError, match="123"):
        tf.finalize_and_render(ses, [123])
    rows = tf.finalize_and_render(ses)
    assert rows.shape == (ses.num_texels, 6) and rows.dtype == np.float32 and rows.flags.c_contiguous
    np.testing.assert_allclose(rows.sum(axis=1), 1.0, atol=1e-4)
    with pytest.raises(RuntimeError):
        tf.finalize_and_render(ses, [0])
    ses = _fresh(scene_dir)
    for fid in (0, 3):
        tf.add_frame(ses, fid, scene_dir[1][fid])
    labels, rows = tf.finalize_and_render(ses, [3, 0])
    assert len(labels) == 2 and all(im.shape == (48, 64) and im.dtype == np.int32 for im in labels)


def test_session_matches_library_pipeline(scene_dir):
    # criterion 11 analogue: the session decode-equals the library calls in the same order
    ses = _fresh(scene_dir)
    for fid in range(8):
        tf.add_frame(ses, fid, scene_dir[1][fid])
    labels, rows = tf.finalize_and_render(ses, list(range(8)))
    mesh = tf.load_mesh(scene_dir[0] / "mesh.ply")
    frames = tf.load_trajectory(scene_dir[0] / "trajectory.txt")
    layout = build_texel_layout(mesh, compute_worst_case_areas(mesh, frames), 0.2)
    tex = init_texture(layout, 6, "mul")
    for fr in frames:
        ids = rasterize(mesh, layout, fr)
        accumulate_frame(tex, ids, scene_dir[1][fr.frame_id], compute_pixel_weights(ids, "images_iid"))
    finalize(tex)
    np.testing.assert_allclose(rows, tex.rows, atol=1e-6)
    lab = texel_argmax(tex)
    for fr, img in zip(frames, labels):
        ids = rasterize(mesh, layout, fr)
        want = render_labels(lab, layout, ids, fallback=scene_dir[1][fr.frame_id].argmax(axis=2).astype(np.int32))
        np.testing.assert_array_equal(img, want)


def test_criterion_11_session_matches_cli(scene_dir, tmp_path):
    # bindings/tests/test_session.py:182-212: session-driven fusion equals the
    # fuse command (texture rows and label images), frames in ascending order
    from paper_2111_11103_b200.cli import main as cli_main
    from paper_2111_11103_b200.formats import read_texture, write_probability_image
    from paper_2111_11103_b200.renderback import read_label_png

    pred = tmp_path / "probs"
    pred.mkdir()
    for fid, p in scene_dir[1].items():
        write_probability_image(pred / ("%d.smpb" % fid), p)
    out = tmp_path / "cli"
    code = cli_main(["fuse", "mesh=%s" % (scene_dir[0] / "mesh.ply"), "trajectory=%s" % (scene_dir[0] / "trajectory.txt"),
                     "predictions=%s" % pred, "classes=6", "gamma=0.2", "aggregator=mul", "weights=images_iid",
                     "deterministic=true", "output=%s" % out])
    assert code == 0
    ids = [f.frame_id for f in tf.load_trajectory(scene_dir[0] / "trajectory.txt")]
    ses = _fresh(scene_dir)
    for fid in ids:
        tf.add_frame(ses, fid, scene_dir[1][fid])
    labels, rows = tf.finalize_and_render(ses, ids)
    cli_rows = read_texture(out / "texture.smtx")[1]
    np.testing.assert_array_equal(rows, cli_rows)
    for fid, img in zip(ids, labels):
        np.testing.assert_array_equal(img, read_label_png(out / "labels" / ("%d.png" % fid)))

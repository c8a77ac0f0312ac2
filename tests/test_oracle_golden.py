"""Pin the CPU oracle against fixtures produced by the reference itself.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py,
which imports the reference package; these tests need only numpy + the
oracle library, so they run on the CPU box and on the GPU box alike.
"""

import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def raster_cases():
    return np.load(os.path.join(GOLD, "raster_cases.npz"))


@pytest.fixture(scope="module")
def cfg1():
    return np.load(os.path.join(GOLD, "cfg1.npz"))


def _case_names(z):
    return [str(n) for n in z["names"]]


def test_to_camera_bits():
    # BLAS dgemm order fma(z,R2,fma(y,R1,x*R0))+t reproduces points @ R.T + t
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 7, 64, 1000, 20000):
        pts = rng.normal(size=(n, 3)) * 3
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        t = rng.normal(size=3)
        cam = np.concatenate([q.reshape(-1), t, [1, 1, 0, 0]])
        np.testing.assert_array_equal(O.to_camera(pts, cam), pts @ q.T + t)


def test_oracle_rasterizer_matches_reference_cases(raster_cases):
    z = raster_cases
    for name in _case_names(z):
        W, H = (int(x) for x in z[name + "/wh"])
        for f, cam in enumerate(z[name + "/cams"]):
            out = O.rasterize(z[name + "/verts"], z[name + "/tris"], z[name + "/steps"],
                              z[name + "/origins"], cam, W, H)
            np.testing.assert_array_equal(out["triangle"], z[name + "/tri"][f], err_msg=name)
            np.testing.assert_array_equal(out["texel"], z[name + "/texel"][f], err_msg=name)
            if name + "/depth" in z:
                # bit-exact float planes (array_equal compares values incl. inf)
                np.testing.assert_array_equal(out["depth"], z[name + "/depth"][f], err_msg=name)
                cov = out["triangle"] >= 0
                np.testing.assert_array_equal(out["u"][cov], z[name + "/u"][f][cov], err_msg=name)
                np.testing.assert_array_equal(out["v"][cov], z[name + "/v"][f][cov], err_msg=name)


def test_golden_cases_cover_edge_conditions(raster_cases):
    z = raster_cases
    names = _case_names(z)
    assert any(n.startswith("clip") for n in names)
    # the chain case really has multi-surface ties, and the coplanar case picks the lower id
    assert (z["coplanar/tri"][0][z["coplanar/tri"][0] >= 0] <= 1).all()
    assert (z["chain/tri"][0] >= 0).sum() > 100


def test_oracle_rasterizer_cfg1(cfg1):
    z = cfg1
    W, H = (int(x) for x in z["wh"])
    for f, cam in enumerate(z["cams"]):
        out = O.rasterize(z["verts"], z["tris"], z["steps"], z["origins"], cam, W, H, want_uv=False)
        np.testing.assert_array_equal(out["triangle"], z["tri"][f])
        np.testing.assert_array_equal(out["texel"], z["texel"][f])


def test_oracle_rasterizer_cfg2_full_frame():
    z = np.load(os.path.join(GOLD, "cfg2_frame.npz"))
    from paper_2111_11103_b200.synth import make_room
    from paper_2111_11103_b200.geometry import uv_origins
    verts, tris = make_room((6.0, 5.0, 3.0), 158)
    assert len(tris) == int(z["n_tris"])
    assert float(verts.sum()) == float(z["verts_sum"])
    steps = np.ones(len(tris), np.int32)
    out = O.rasterize(verts, tris, steps, uv_origins(verts, tris), z["cam"], 640, 480, want_uv=False)
    np.testing.assert_array_equal(out["triangle"], z["tri"])
    np.testing.assert_array_equal(out["texel"], z["texel"])
    assert float(out["depth"][out["triangle"] >= 0].sum()) == float(z["depth_sum"])


def test_oracle_layout_cfg1(cfg1):
    offsets, total = O.layout_arrays(cfg1["steps"])
    np.testing.assert_array_equal(offsets, cfg1["offsets"])
    assert total == int(cfg1["total_texels"])


@pytest.mark.parametrize("agg", O.AGGREGATORS)
@pytest.mark.parametrize("wm", ["images_iid", "pixels_iid"])
def test_oracle_fusion_cfg1_bitexact(cfg1, agg, wm):
    z = cfg1
    key = "%s_%s" % (agg, wm)
    c = int(z["num_classes"])
    n_x = int(z["total_texels"])
    probs = cfg1_probs(z)
    accum = np.zeros((n_x, c))
    counts = np.zeros(n_x, np.int64)
    for f in range(len(z["cams"])):
        w = O.compute_pixel_weights(z["tri"][f], z["texel"][f], wm)
        if f == 0 and key + "/weights0" in z:
            np.testing.assert_array_equal(w, z[key + "/weights0"])
        O.accumulate_frame(accum, counts, z["offsets"], z["tri"][f], z["texel"][f], probs[f], w, agg)
    np.testing.assert_array_equal(counts, z[key + "/counts"])
    np.testing.assert_array_equal(accum, z[key + "/accum"])
    rows, unobs = O.finalize(accum, counts, agg)
    np.testing.assert_array_equal(rows, z[key + "/rows"])
    np.testing.assert_array_equal(unobs, z[key + "/unobserved"])
    labels = O.texel_argmax(rows, unobs)
    np.testing.assert_array_equal(labels, z[key + "/labels"])
    if key + "/rendered" in z:
        for f in range(len(z["cams"])):
            fb = probs[f].argmax(axis=2).astype(np.int32)
            out = O.render_labels(labels, z["offsets"], z["tri"][f], z["texel"][f], fallback=fb)
            np.testing.assert_array_equal(out, z[key + "/rendered"][f])


@pytest.mark.parametrize("agg", O.AGGREGATORS)
def test_oracle_c_fuse_matches_numpy(cfg1, agg):
    z = cfg1
    c = int(z["num_classes"])
    n_x = int(z["total_texels"])
    probs = cfg1_probs(z)
    W, H = (int(x) for x in z["wh"])
    accum, counts = O.fuse_frames_c(z["verts"], z["tris"], z["steps"], z["origins"], z["offsets"], n_x,
                                    z["cams"], W, H, probs, agg, "images_iid", nthreads=2)
    ref = z["%s_images_iid/accum" % agg]
    np.testing.assert_array_equal(counts, z["%s_images_iid/counts" % agg])
    np.testing.assert_allclose(accum, ref, rtol=1e-12, atol=1e-12)
    rows, unobs, labels = O.finalize_c(accum, counts, agg)
    np.testing.assert_array_equal(unobs, z["%s_images_iid/unobserved" % agg])
    np.testing.assert_allclose(rows, z["%s_images_iid/rows" % agg], atol=1e-6)


def cfg1_probs(z):
    from paper_2111_11103_b200.synth import NoiseModel, corrupt
    model = NoiseModel("flip", epsilon=0.3, q=0.8, seed=1)
    c = int(z["num_classes"])
    return [corrupt(z["gt"][f].astype(np.int32), model, c, f) for f in range(len(z["cams"]))]


def test_oracle_areas_and_layout_cfg1(cfg1):
    z = cfg1
    W, H = (int(x) for x in z["wh"])
    sizes = np.tile([W, H], (len(z["cams"]), 1))
    areas = O.worst_case_areas(z["verts"], z["tris"], z["cams"], sizes)
    np.testing.assert_array_equal(areas, z["areas"])
    np.testing.assert_array_equal(O.build_steps(areas, 0.2), z["steps"])


def test_oracle_areas_cfg2_golden():
    """The C restatement of compute_worst_case_areas on the configs[1] mesh (300k triangles,
    4 cameras) equals the reference's output bit for bit (fixture: make_golden.py cfg2areas)."""
    import oracle as O
    from paper_2111_11103_b200.synth import make_room

    z = np.load(os.path.join(GOLD, "cfg2_areas.npz"))
    v, t = make_room((6.0, 5.0, 3.0), 158)
    sizes = np.tile(np.array([[640, 480]], np.int32), (len(z["cams"]), 1))
    areas = O.worst_case_areas(v, t, z["cams"], sizes)
    np.testing.assert_array_equal(areas, z["areas"])

"""Host-side logic of the drop-in API (no GPU): data model, layout, config
parsing, I/O and validation order, checked against the reference goldens and
the reference's own test expectations (tests/test_geometry.py,
tests/test_fusion.py, tests/test_meshio.py, bindings/tests/test_session.py)."""

import math
import os

import numpy as np
import pytest

from paper_2111_11103_b200 import (CapacityError, DataError, Mesh, build_texel_layout, compute_pixel_weights,
                                   init_texture, load_mesh, load_trajectory, parse_weight_mode, save_ply,
                                   save_trajectory, texel_count, texel_id, texture_nbytes, uniform_layout)
from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics, MAX_STEPS, uv_origins
from paper_2111_11103_b200.rasterizer import IdImage
from paper_2111_11103_b200.synth import (NoiseModel, corrupt, make_cube, make_icosphere, make_orbit_trajectory,
                                         make_room)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def strip_mesh(n):
    verts, tris = [], []
    for k in range(n):
        verts += [(2.0 * k, 0, 0), (2.0 * k + 1, 0, 0), (2.0 * k, 1, 0)]
        tris.append((3 * k, 3 * k + 1, 3 * k + 2))
    return Mesh.from_arrays(np.array(verts, float), np.array(tris))


def test_synthetic_room_equals_reference_mesh():
    z = np.load(os.path.join(GOLD, "cfg1.npz"))
    v, t = make_room((6.0, 5.0, 3.0), 32)
    np.testing.assert_array_equal(v, z["verts"])
    np.testing.assert_array_equal(t, z["tris"])
    np.testing.assert_array_equal(uv_origins(v, t), z["origins"])


def test_layout_from_reference_areas_matches_reference_layout():
    z = np.load(os.path.join(GOLD, "cfg1.npz"))
    mesh = Mesh(z["verts"], z["tris"])
    layout = build_texel_layout(mesh, z["areas"], 0.2)
    np.testing.assert_array_equal(layout.steps, z["steps"])
    np.testing.assert_array_equal(layout.offsets, z["offsets"])
    assert layout.total_texels == int(z["total_texels"])


def test_texel_id_bijection():
    # acceptance criterion 1 (test_acceptance.py:53-65)
    for s in range(1, 65):
        ids = sorted(texel_id(s, (i + 0.5) / s, (j + 0.5) / s) for i in range(s) for j in range(i + 1))
        assert ids == list(range((s * s + s) // 2))
    assert texel_count(6) == 21


def test_layout_rules():
    mesh = strip_mesh(5)
    lay = build_texel_layout(mesh, np.array([400.0, 0.0, 25.0, 10000.0, 1.0]), 0.2)
    assert lay.steps.tolist() == [4, 1, 1, 20, 1]
    np.testing.assert_array_equal(np.diff(lay.offsets), lay.texel_counts()[:-1])
    assert build_texel_layout(strip_mesh(1), np.array([1e9]), 1.0).steps[0] == MAX_STEPS
    with pytest.raises(ValueError):
        build_texel_layout(mesh, np.zeros(5), -0.1)
    with pytest.raises(DataError):
        build_texel_layout(mesh, np.zeros(3), 0.2)
    assert uniform_layout(strip_mesh(4), 3).total_texels == 24
    rng = np.random.default_rng(3)
    areas = rng.uniform(1, 3000, 50)
    for g in (0.1, 0.3, 0.9):
        s1 = build_texel_layout(strip_mesh(50), areas, g).steps
        s2 = build_texel_layout(strip_mesh(50), 2 * areas, g).steps
        assert (s2 >= s1).all() and (s2 <= np.ceil(math.sqrt(2.0) * s1)).all()


def test_mesh_validation():
    with pytest.raises(DataError):
        Mesh(np.zeros((3, 3)), np.array([[0, 1, 5]]))
    m = Mesh.from_arrays(np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0.0], [0, 1, 0]]), np.array([[0, 1, 2], [0, 1, 3]]))
    assert m.num_triangles == 1 and m.dropped_degenerate == 1
    with pytest.raises(DataError):
        CameraFrame(0, Intrinsics(1, 1, 0, 0, 4, 4), np.ones((3, 3)), np.zeros(3))
    with pytest.raises(DataError):
        Intrinsics(0, 1, 0, 0, 4, 4)


def test_parse_weight_mode_forms():
    assert parse_weight_mode("pixels_iid") == ("pixels_iid", None)
    assert parse_weight_mode("images_iid") == ("images_iid", None)
    assert parse_weight_mode("blend:0.25") == ("blend", 0.25)
    assert parse_weight_mode("blend(0.25)") == ("blend", 0.25)
    for bad in ("blend", "blend:1.5", "blend:-0.1", "votes"):
        with pytest.raises(ValueError):
            parse_weight_mode(bad)


def test_texture_validation_precedes_device_allocation():
    layout = uniform_layout(strip_mesh(1))
    with pytest.raises(ValueError):
        init_texture(layout, 1, "sum")
    with pytest.raises(ValueError):
        init_texture(layout, 3, "median")
    big = build_texel_layout(strip_mesh(13), np.full(13, 4.0e9), 5.0)
    need = texture_nbytes(big.total_texels, 40)
    with pytest.raises(CapacityError) as err:
        init_texture(big, 40, "sum", memory_budget=2 ** 30)
    assert str(need) in str(err.value) and str(2 ** 30) in str(err.value)
    ids = IdImage(0, 2, 1, triangle=np.array([[0, 0]]), texel=np.array([[0, 0]]))
    with pytest.raises(ValueError):
        compute_pixel_weights(ids, "votes")
    with pytest.raises(ValueError):
        compute_pixel_weights(ids, "blend", None)


def test_ply_obj_and_trajectory_round_trips(tmp_path):
    mesh = make_icosphere(1.0, 1)
    for binary in (True, False):
        p = tmp_path / ("m_%d.ply" % binary)
        save_ply(p, mesh, binary=binary)
        back = load_mesh(p)
        np.testing.assert_array_equal(back.triangles, mesh.triangles)
        # binary stores float32 exactly; ascii uses %g like the reference writer (meshio.py:251)
        np.testing.assert_allclose(back.vertices, mesh.vertices.astype(np.float32), rtol=0,
                                   atol=0 if binary else 1e-5)
    obj = tmp_path / "q.obj"
    obj.write_text("v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n")
    assert load_mesh(obj).num_triangles == 2
    intr = Intrinsics(64.0, 64.0, 32.0, 24.0, 64, 48)
    frames = make_orbit_trajectory((0, 0, 0), 3.0, 5, intr, tilt_deg=10.0)
    tp = tmp_path / "traj.txt"
    save_trajectory(tp, frames[::-1])
    back = load_trajectory(tp)
    assert [f.frame_id for f in back] == list(range(5))
    np.testing.assert_array_equal(back[2].rotation, frames[2].rotation)
    with pytest.raises(DataError, match="nowhere.ply"):
        load_mesh(tmp_path / "nowhere.ply")
    bad = tmp_path / "bad.txt"
    bad.write_text("0 1 2 3\n")
    with pytest.raises(DataError, match="19 fields"):
        load_trajectory(bad)


def test_session_errors_name_missing_paths(tmp_path):
    from paper_2111_11103_b200 import open_session

    with pytest.raises(DataError, match="nowhere.ply"):
        open_session(tmp_path / "nowhere.ply", tmp_path / "t.txt", 0.2, "mul", "images_iid", 6)


def test_noise_model_is_frame_keyed():
    gt = np.full((4, 5), 2, dtype=np.int32)
    gt[0, 0] = -1
    m = NoiseModel("flip", 0.3, 0.8, seed=9)
    a = corrupt(gt, m, 6, 3)
    np.testing.assert_array_equal(a, corrupt(gt, m, 6, 3))
    assert not np.array_equal(a, corrupt(gt, m, 6, 4))
    np.testing.assert_allclose(a.sum(axis=2), 1.0, atol=1e-6)
    np.testing.assert_allclose(a[0, 0], 1.0 / 6)
    assert make_cube().num_triangles == 12

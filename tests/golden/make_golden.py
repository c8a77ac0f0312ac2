"""Generate the golden fixtures that pin the oracle (and, through it, the GPU path).

Run in the build container only — it imports the *reference* package
read-only from /root/reference/pkg/src (that tree does not exist on the GPU
box, so nothing at test time imports it; the tests read the .npz files this
script writes):

    python tests/golden/make_golden.py

Every array stored here is an output of the reference's own functions
(rasterize, compute_worst_case_areas, build_texel_layout, compute_pixel_weights,
accumulate_frame, finalize, texel_argmax, render_labels) on seeded inputs.
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

import texelfuse as tf  # noqa: E402
from texelfuse import synthgen  # noqa: E402
from texelfuse.rasterizer import rasterize  # noqa: E402


def cam16(frame):
    return np.concatenate([frame.rotation.reshape(-1), frame.translation.reshape(-1),
                           [frame.fx, frame.fy, frame.cx, frame.cy]]).astype(np.float64)


def frontal(width=64, height=64, fx=None, frame_id=0, translation=(0.0, 0.0, 0.0)):
    fx = float(width) if fx is None else fx
    intr = tf.Intrinsics(fx=fx, fy=fx, cx=width / 2.0, cy=height / 2.0, width=width, height=height)
    return tf.CameraFrame(frame_id=frame_id, intrinsics=intr, rotation=np.eye(3),
                          translation=np.asarray(translation, dtype=np.float64))


def random_scene(seed):
    # test_acceptance.py:163-174 (criterion 4 scene generator)
    rng = np.random.default_rng(seed)
    m = int(rng.integers(5, 51))
    centers = np.stack([rng.uniform(-1.2, 1.2, m), rng.uniform(-1.2, 1.2, m),
                        rng.uniform(1.5, 4.0, m)], axis=1)
    verts = (centers[:, None, :] + rng.normal(scale=0.45, size=(m, 3, 3))).reshape(-1, 3)
    verts[:, 2] = np.maximum(verts[:, 2], 0.3)
    return tf.Mesh.from_arrays(verts, np.arange(3 * m).reshape(m, 3))


def clip_scene(seed):
    # triangles straddling / behind the near plane, to exercise the clip + fan path
    rng = np.random.default_rng(1000 + seed)
    m = 40
    centers = np.stack([rng.uniform(-0.6, 0.6, m), rng.uniform(-0.6, 0.6, m),
                        rng.uniform(-0.5, 1.5, m)], axis=1)
    verts = (centers[:, None, :] + rng.normal(scale=0.6, size=(m, 3, 3))).reshape(-1, 3)
    return tf.Mesh.from_arrays(verts, np.arange(3 * m).reshape(m, 3))


def chain_scene():
    # near-coplanar stacks within the 1e-9 m tie tolerance, drawn far-to-near and
    # near-to-far: exercises the sequential (non-transitive) depth-tie fold
    quads = []
    for k, dz in enumerate([1.5e-9, 0.7e-9, 0.0, 5e-10, 5e-9, 2.2e-9]):
        z = 2.0 + dz
        h = 0.5 - 0.03 * k
        quads.append(np.array([[-h, -h, z], [h, -h, z], [h, h, z], [-h, h, z]]))
    verts = np.concatenate(quads)
    tris = []
    for k in range(len(quads)):
        b = 4 * k
        tris += [(b, b + 1, b + 2), (b, b + 2, b + 3)]
    return tf.Mesh.from_arrays(verts, np.array(tris, dtype=np.int32))


def vertex_pixel_mesh(depths):
    # test_rasterizer.py:107-114
    screen = [(10.5, 10.5), (50.5, 12.5), (12.5, 52.5)]
    verts = [((px - 32.0) / 64.0 * z, (py - 32.0) / 64.0 * z, z) for (px, py), z in zip(screen, depths)]
    return tf.Mesh.from_arrays(np.array(verts), np.array([[0, 1, 2]]))


def raster_cases():
    cases = []  # (name, mesh, layout, [frames], store_float_planes)
    for seed in range(12):
        mesh = random_scene(seed)
        cases.append(("random%d" % seed, mesh, tf.uniform_layout(mesh, 1 + seed % 4),
                      [frontal(64, 64, 64.0)], True))
    for seed in range(4):
        mesh = clip_scene(seed)
        cases.append(("clip%d" % seed, mesh, tf.uniform_layout(mesh, 3),
                      [frontal(64, 64, 64.0)], True))
    cube = synthgen.make_cube()
    intr = frontal(64, 48, 48.0).intrinsics
    cases.append(("cube_orbit", cube.mesh, tf.uniform_layout(cube.mesh, 6),
                  synthgen.make_orbit_trajectory((0, 0, 0), 3.0, 6, intr, tilt_deg=20.0), True))
    ico = synthgen.make_icosphere(radius=1.0, level=1)
    cases.append(("icosphere", ico, tf.uniform_layout(ico, 4),
                  [frontal(80, 60, 70.0, 3, (0.0, 0.0, 3.0))], True))
    cases.append(("chain", chain_scene(), tf.uniform_layout(chain_scene(), 2),
                  [frontal(64, 64, 64.0)], True))
    for k, d in enumerate([(1.0, 2.0, 3.0), (2.0, 1.0, 3.0), (1.0, 3.0, 2.0)]):
        mesh = vertex_pixel_mesh(d)
        cases.append(("vertexpix%d" % k, mesh, tf.uniform_layout(mesh, 5 + 2 * k),
                      [frontal(64, 64, 64.0)], True))
    one = tf.Mesh.from_arrays(np.array([[-0.4, -0.4, 2.0], [0.4, -0.4, 2.0], [0.4, 0.4, 2.0], [-0.4, 0.4, 2.0]]),
                              np.array([[0, 1, 2], [0, 2, 3]]))
    copl = tf.Mesh.from_arrays(np.vstack([one.vertices, one.vertices]),
                               np.vstack([one.triangles, one.triangles + 4]))
    cases.append(("coplanar", copl, tf.uniform_layout(copl), [frontal(64, 64, 64.0)], True))
    return cases


def write_raster_cases(path):
    out = {}
    names = []
    for name, mesh, layout, frames, store in raster_cases():
        names.append(name)
        out[name + "/verts"] = mesh.vertices
        out[name + "/tris"] = mesh.triangles
        out[name + "/steps"] = layout.steps
        out[name + "/origins"] = layout.origins
        out[name + "/offsets"] = layout.offsets
        cams, tri, tex, dep, uu, vv = [], [], [], [], [], []
        for fr in frames:
            ids = rasterize(mesh, layout, fr)
            cams.append(cam16(fr))
            tri.append(ids.triangle)
            tex.append(ids.texel)
            dep.append(ids.depth)
            uu.append(ids.u)
            vv.append(ids.v)
        out[name + "/cams"] = np.stack(cams)
        out[name + "/wh"] = np.array([frames[0].width, frames[0].height])
        out[name + "/tri"] = np.stack(tri)
        out[name + "/texel"] = np.stack(tex)
        if store:
            out[name + "/depth"] = np.stack(dep)
            out[name + "/u"] = np.stack(uu)
            out[name + "/v"] = np.stack(vv)
    out["names"] = np.array(names)
    np.savez_compressed(path, **out)


def cfg1_scene():
    """BASELINE.json configs[0]: room tess=32 (12,288 tris), 20 frames 160x120, c=13."""
    scene = synthgen.make_room(size=(6.0, 5.0, 3.0), tess=32, num_classes=13)
    intr = tf.Intrinsics(fx=160.0, fy=160.0, cx=80.0, cy=60.0, width=160, height=120)
    frames = synthgen.make_orbit_trajectory((0, 0, 0), 1.0, 20, intr, tilt_deg=20.0)
    return scene, frames


def write_cfg1(path):
    t0 = time.time()
    scene, frames = cfg1_scene()
    mesh = scene.mesh
    c = scene.num_classes
    areas = tf.compute_worst_case_areas(mesh, frames)
    layout = tf.build_texel_layout(mesh, areas, 0.2)
    model = tf.NoiseModel("flip", epsilon=0.3, q=0.8, seed=1)
    out = {"verts": mesh.vertices, "tris": mesh.triangles, "areas": areas,
           "steps": layout.steps, "origins": layout.origins, "offsets": layout.offsets,
           "total_texels": np.int64(layout.total_texels),
           "cams": np.stack([cam16(f) for f in frames]),
           "wh": np.array([160, 120]), "num_classes": np.int64(c)}
    tri, tex, gts = [], [], []
    ids_all = []
    for fr in frames:
        ids = rasterize(mesh, layout, fr)
        ids_all.append(ids)
        tri.append(ids.triangle)
        tex.append(ids.texel)
        gts.append(tf.render_ground_truth(scene, fr, ids))
    out["tri"] = np.stack(tri)
    out["texel"] = np.stack(tex)
    out["gt"] = np.stack(gts).astype(np.int8)
    probs = [tf.corrupt(g, model, c, fr.frame_id) for g, fr in zip(gts, frames)]
    for agg in ("sum", "mul", "maxsum"):
        for wm in ("images_iid", "pixels_iid"):
            tex_ = tf.init_texture(layout, c, agg)
            for ids, p in zip(ids_all, probs):
                w = tf.compute_pixel_weights(ids, wm)
                tf.accumulate_frame(tex_, ids, p, w)
            key = "%s_%s" % (agg, wm)
            out[key + "/accum"] = tex_.accum.copy()
            out[key + "/counts"] = tex_.counts.copy()
            tf.finalize(tex_)
            out[key + "/rows"] = tex_.rows
            out[key + "/unobserved"] = tex_.unobserved
            labels = tf.texel_argmax(tex_)
            out[key + "/labels"] = labels
            if agg == "sum" and wm == "images_iid":
                rendered = []
                for ids, p in zip(ids_all, probs):
                    fb = p.argmax(axis=2).astype(np.int32)
                    rendered.append(tf.render_labels(labels, layout, ids, fallback=fb))
                out[key + "/rendered"] = np.stack(rendered).astype(np.int8)
                out[key + "/weights0"] = tf.compute_pixel_weights(ids_all[0], wm)
    np.savez_compressed(path, **out)
    print("cfg1 golden in %.1f s" % (time.time() - t0))


def write_cfg2_frame(path):
    """One full-size frame of the BASELINE configs[1] mesh (300k tris, 640x480)."""
    t0 = time.time()
    scene = synthgen.make_room(size=(6.0, 5.0, 3.0), tess=158, num_classes=40)
    mesh = scene.mesh
    layout = tf.uniform_layout(mesh, 1)
    intr = tf.Intrinsics(fx=577.87, fy=577.87, cx=319.5, cy=239.5, width=640, height=480)
    rot, trans = synthgen.look_at((1.1, -0.7, 0.2), (-2.0, 1.5, -0.4))
    fr = tf.CameraFrame(frame_id=0, intrinsics=intr, rotation=rot, translation=trans)
    ids = rasterize(mesh, layout, fr)
    np.savez_compressed(path, cam=cam16(fr), wh=np.array([640, 480]), tri=ids.triangle,
                        texel=ids.texel, depth_sum=np.float64(ids.depth[ids.covered].sum()),
                        n_tris=np.int64(mesh.num_triangles), verts_sum=np.float64(mesh.vertices.sum()))
    print("cfg2 frame golden in %.1f s" % (time.time() - t0))


def write_cfg2_areas(path):
    """compute_worst_case_areas + build_texel_layout (geometry.py:257-380) on the BASELINE
    configs[1] mesh over 4 seeded in-room cameras (paper_2111_11103_b200.synth's
    random_room_trajectory poses), at gamma 0.2 and 1.0."""
    t0 = time.time()
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2111_11103_b200.synth import random_room_trajectory, scannet_intrinsics

    scene = synthgen.make_room(size=(6.0, 5.0, 3.0), tess=158, num_classes=40)
    mesh = scene.mesh
    intr = tf.Intrinsics(fx=577.87, fy=577.87, cx=319.5, cy=239.5, width=640, height=480)
    poses = random_room_trajectory(4, scannet_intrinsics(), seed=21)
    frames = [tf.CameraFrame(frame_id=k, intrinsics=intr, rotation=p.rotation, translation=p.translation)
              for k, p in enumerate(poses)]
    areas = tf.compute_worst_case_areas(mesh, frames)
    out = {"cams": np.stack([cam16(f) for f in frames]), "areas": areas}
    for gamma in (0.2, 1.0):
        lay = tf.build_texel_layout(mesh, areas, gamma)
        out["steps_%g" % gamma] = lay.steps.astype(np.int32)
        out["origins_%g" % gamma] = lay.origins.astype(np.int8)
        out["total_%g" % gamma] = np.int64(lay.total_texels)
    np.savez_compressed(path, **out)
    print("cfg2 areas golden in %.1f s" % (time.time() - t0))


if __name__ == "__main__":
    what = sys.argv[1:] or ["raster", "cfg1", "cfg2", "cfg2areas"]
    if "raster" in what:
        write_raster_cases(os.path.join(HERE, "raster_cases.npz"))
    if "cfg1" in what:
        write_cfg1(os.path.join(HERE, "cfg1.npz"))
    if "cfg2" in what:
        write_cfg2_frame(os.path.join(HERE, "cfg2_frame.npz"))
    if "cfg2areas" in what:
        write_cfg2_areas(os.path.join(HERE, "cfg2_areas.npz"))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))

"""Synthetic scenes, trajectories and probability maps for tests and benchmarks.

The mesh builders and noise model produce the same numbers as the
reference's fixture source (texelfuse/synthgen.py): make_room (:116-158),
make_cube (:82-113), make_icosphere (:161-198), look_at (:238-257),
make_orbit_trajectory (:260-291) and corrupt (:313-346, Philox keyed on
(seed, frame_id)).  random_room_trajectory and softmax maps implement the
BASELINE configs[1] workload.  None of this is on the hot path.
"""

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError
from .geometry import CameraFrame, Intrinsics, Mesh


def _grid_face(origin, eu, ev, tess, base):
    o = np.asarray(origin, dtype=np.float64)
    eu = np.asarray(eu, dtype=np.float64)
    ev = np.asarray(ev, dtype=np.float64)
    verts = [o + eu * (i / tess) + ev * (j / tess) for i in range(tess + 1) for j in range(tess + 1)]
    tris = []
    for i in range(tess):
        for j in range(tess):
            a = base + i * (tess + 1) + j
            b = a + tess + 1
            tris.append((a, b, b + 1))
            tris.append((a, b + 1, a + 1))
    return verts, tris


def make_room(size=(6.0, 5.0, 3.0), tess=4):
    """Inward-facing tessellated box: 12*tess^2 triangles.  Returns (vertices, triangles)
    with face order floor, ceiling, +x, -x, +y, -y (synthgen.py:116-158)."""
    if tess < 1:
        raise ConfigError("tess must be >= 1")
    hx, hy, hz = (float(s) / 2.0 for s in size)
    ex, ey, ez = (2 * hx, 0, 0), (0, 2 * hy, 0), (0, 0, 2 * hz)
    faces = [((-hx, -hy, -hz), ex, ey), ((-hx, -hy, hz), ey, ex), ((hx, -hy, -hz), ey, ez),
             ((-hx, -hy, -hz), ez, ey), ((-hx, hy, -hz), ex, ez), ((-hx, -hy, -hz), ez, ex)]
    verts, tris = [], []
    for origin, eu, ev in faces:
        v, t = _grid_face(origin, eu, ev, tess, len(verts))
        verts += v
        tris += t
    return np.array(verts, dtype=np.float64), np.array(tris, dtype=np.int32)


def make_furnished_room(size=(6.0, 5.0, 3.0), tess=4, num_boxes=10, box_tess=6, seed=0):
    """make_room plus `num_boxes` closed, tessellated boxes ("furniture") standing
    on the floor, each 12 * box_tess^2 triangles (SURVEY §7 hard part 9: the bare
    room seen from inside has no overdraw; the boxes give occlusion, so pixels
    with several covering triangles and the depth test).  Boxes may overlap each
    other; they stay inside the central 80 % of the floor.  Returns (vertices,
    triangles); the room's triangles come first."""
    v, t = make_room(size, tess)
    rng = np.random.default_rng(seed)
    hx, hy, hz = (float(s) / 2.0 for s in size)
    verts, tris = [v], [t]
    nv = len(v)
    for _ in range(num_boxes):
        w, d, h = rng.uniform(0.3, 1.2), rng.uniform(0.3, 1.2), rng.uniform(0.3, 1.1)
        x0 = rng.uniform(-0.8 * hx, 0.8 * hx - w)
        y0 = rng.uniform(-0.8 * hy, 0.8 * hy - d)
        z0 = -hz + 1e-3  # just above the floor (no coplanar faces with it)
        ex, ey, ez = (w, 0, 0), (0, d, 0), (0, 0, h)
        faces = [((x0, y0, z0), ey, ex), ((x0, y0, z0 + h), ex, ey), ((x0 + w, y0, z0), ey, ez),
                 ((x0, y0, z0), ez, ey), ((x0, y0 + d, z0), ez, ex), ((x0, y0, z0), ex, ez)]
        for origin, eu, ev in faces:
            fv, ft = _grid_face(origin, eu, ev, box_tess, nv)
            verts.append(np.array(fv, dtype=np.float64))
            tris.append(np.array(ft, dtype=np.int32))
            nv += len(fv)
    return np.concatenate(verts), np.concatenate(tris).astype(np.int32)


def room_face_labels(tess, num_classes):
    per = 2 * tess * tess
    return (np.repeat(np.arange(6), per) % num_classes).astype(np.int32)


def make_room_mesh(size=(6.0, 5.0, 3.0), tess=4):
    v, t = make_room(size, tess)
    return Mesh.from_arrays(v, t)


def make_cube(size=2.0):
    """12-triangle axis-aligned cube; face classes +x -x +y -y +z -z (synthgen.py:82-113)."""
    h = size / 2.0
    corners = np.array([[sx, sy, sz] for sx in (-h, h) for sy in (-h, h) for sz in (-h, h)], dtype=np.float64)
    quads = [(4, 6, 7, 5), (0, 1, 3, 2), (2, 3, 7, 6), (0, 4, 5, 1), (1, 5, 7, 3), (0, 2, 6, 4)]
    tris = []
    for a, b, c, d in quads:
        tris += [(a, b, c), (a, c, d)]
    return Mesh.from_arrays(corners, np.array(tris, dtype=np.int32))


def make_icosphere(radius=1.0, level=2):
    """Subdivided icosahedron on the sphere (synthgen.py:161-198)."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    raw = np.array([[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0], [0, -1, phi], [0, 1, phi],
                    [0, -1, -phi], [0, 1, -phi], [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]],
                   dtype=np.float64)
    verts = [v / np.linalg.norm(v) for v in raw]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                p = verts[a] + verts[b]
                verts.append(p / np.linalg.norm(p))
                cache[key] = len(verts) - 1
            return cache[key]

        nxt = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nxt
    return Mesh.from_arrays(np.array(verts, dtype=np.float64) * radius, np.array(faces, dtype=np.int32))


def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """World→camera (R, t) for x right / y down / z forward (synthgen.py:238-257)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    n = np.linalg.norm(fwd)
    if n == 0.0:
        raise ValueError("eye and target coincide")
    z = fwd / n
    up = np.asarray(up, dtype=np.float64)
    if abs(float(np.dot(z, up)) / np.linalg.norm(up)) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    x = np.cross(z, up)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])
    return R, -R @ eye


def make_orbit_trajectory(center, radius, num_frames, intrinsics, tilt_deg=0.0, start_id=0):
    """Cameras on a circle looking at ``center`` (synthgen.py:260-291)."""
    if num_frames < 1:
        raise ConfigError("need at least one frame")
    if radius <= 0.0:
        raise ConfigError("radius must be positive")
    center = np.asarray(center, dtype=np.float64)
    tilt = math.radians(tilt_deg)
    out = []
    for k in range(num_frames):
        th = 2.0 * math.pi * k / num_frames
        el = tilt * math.sin(2.0 * th)
        eye = center + radius * np.array([math.cos(el) * math.cos(th), math.cos(el) * math.sin(th), math.sin(el)])
        R, t = look_at(eye, center)
        out.append(CameraFrame(frame_id=start_id + k, intrinsics=intrinsics, rotation=R, translation=t))
    return out


def scannet_intrinsics():
    """640x480 ScanNet-like pinhole used by BASELINE configs[1]."""
    return Intrinsics(fx=577.87, fy=577.87, cx=319.5, cy=239.5, width=640, height=480)


def random_room_trajectory(num_frames, intrinsics, size=(6.0, 5.0, 3.0), seed=0):
    """Seeded random cameras inside the room: eye ~ U(0.6 * box), yaw ~ U(0, 2pi),
    pitch ~ U(-30, 30) deg, look_at with +z up."""
    rng = np.random.default_rng(seed)
    half = 0.6 * np.asarray(size, dtype=np.float64) / 2.0
    frames = []
    for k in range(num_frames):
        eye = rng.uniform(-half, half)
        yaw = rng.uniform(0.0, 2.0 * math.pi)
        pitch = math.radians(rng.uniform(-30.0, 30.0))
        d = np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch)])
        R, t = look_at(eye, eye + d)
        frames.append(CameraFrame(frame_id=k, intrinsics=intrinsics, rotation=R, translation=t))
    return frames


@dataclass
class NoiseModel:
    """flip / dirichlet prediction noise (synthgen.py:32-56)."""

    kind: str = "flip"
    epsilon: float = 0.3
    q: float = 0.8
    kappa: float = 8.0
    seed: int = 0


def corrupt(gt, model, num_classes, frame_id=0):
    """Noisy (H, W, c) float32 probabilities from labels, Philox keyed on
    (seed, frame_id) (synthgen.py:309-346)."""
    gt = np.asarray(gt)
    c = num_classes
    h, w = gt.shape
    rng = np.random.Generator(np.random.Philox(key=[model.seed, frame_id]))
    known = (gt >= 0) & (gt < c)
    g = np.where(known, gt, 0).astype(np.int64)
    if model.kind == "flip":
        flip_draw = rng.random((h, w))
        wrong_draw = rng.random((h, w))
        wrong = np.minimum((wrong_draw * (c - 1)).astype(np.int64), c - 2)
        wrong += wrong >= g
        chosen = np.where(flip_draw < model.epsilon, wrong, g)
        probs = np.full((h, w, c), (1.0 - model.q) / (c - 1), dtype=np.float32)
        np.put_along_axis(probs, chosen[..., None], np.float32(model.q), axis=2)
    else:
        alpha = np.ones((h, w, c), dtype=np.float64)
        np.put_along_axis(alpha, g[..., None], 1.0 + model.kappa, axis=2)
        draws = rng.standard_gamma(alpha)
        probs = (draws / draws.sum(axis=2, keepdims=True)).astype(np.float32)
    probs[~known] = np.float32(1.0 / c)
    return probs


def softmax_maps(n, height, width, num_classes, seed=0, scale=2.0, device="cuda"):
    """n random softmax(N(0, scale^2)) probability maps (n, H, W, c) float32 on ``device``."""
    import torch

    g = torch.Generator(device=device)
    out = torch.empty((n, height, width, num_classes), dtype=torch.float32, device=device)
    for i in range(n):
        g.manual_seed(1000 * seed + i)
        logits = torch.randn((height, width, num_classes), generator=g, device=device) * scale
        out[i] = torch.softmax(logits, dim=-1)
    return out

"""TEST INFRASTRUCTURE ONLY — NumPy/C restatement of the reference hot path.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/texelfuse).  Inputs are plain arrays so the oracle is
independent of both the reference package and the product package.
"""

import ctypes
import os
import subprocess

import numpy as np

__all__ = [
    "NEAR_PLANE", "DEPTH_TIE", "MUL_CLAMP", "UNKNOWN", "AGGREGATORS", "WEIGHT_MODES",
    "lib", "build", "to_camera", "rasterize", "texel_count", "layout_arrays",
    "compute_pixel_weights", "accumulate_frame", "finalize", "texel_argmax",
    "render_labels", "fuse_frames_c", "finalize_c", "pixel_rows", "worst_case_areas", "build_steps",
]

NEAR_PLANE = 1e-4  # geometry.py:26
DEPTH_TIE = 1e-9  # rasterizer.py:18
MUL_CLAMP = 1e-7  # fusion.py:39
UNKNOWN = -1  # fusion.py:42
AGGREGATORS = ("sum", "maxsum", "mul")  # fusion.py:34
WEIGHT_MODES = ("pixels_iid", "images_iid", "blend")  # fusion.py:35

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int


def build():
    """Compile the C restatement (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.tfo_to_camera.argtypes = [_P, _I64, _P, _P]
        L.tfo_rasterize.argtypes = [_P, _I64, _P, _I64, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P]
        L.tfo_rasterize.restype = _I
        L.tfo_fuse_frames.argtypes = [_P, _I64, _P, _I64, _P, _P, _P, _I64, _I, _P, _I, _I,
                                      _I64, _P, _I, _I, ctypes.c_double, _P, _P, _I]
        L.tfo_fuse_frames.restype = _I
        L.tfo_finalize.argtypes = [_P, _P, _I64, _I, _I, _P, _P, _P]
        L.tfo_worst_case_areas.argtypes = [_P, _I64, _P, _I64, _P, _P, _I64, _P]
        _lib = L
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def texel_count(steps):
    """geometry.py:181-185."""
    s = np.asarray(steps, dtype=np.int64)
    out = (s * s + s) // 2
    return out if out.ndim else int(out)


def layout_arrays(steps):
    """Packed offsets + total texels from per-triangle steps (geometry.py:282-290, 298-305)."""
    counts = texel_count(np.asarray(steps))
    offsets = np.zeros(len(counts), dtype=np.int64)
    if len(counts):
        np.cumsum(counts[:-1], out=offsets[1:])
    return offsets, int(np.sum(counts))


def to_camera(verts, cam16):
    """geometry.py:159-161 with the BLAS FMA order."""
    v = _c(verts, np.float64).reshape(-1, 3)
    cam = _c(cam16, np.float64)
    out = np.empty_like(v)
    lib().tfo_to_camera(_ptr(v), len(v), _ptr(cam), _ptr(out))
    return out


def rasterize(verts, tris, steps, origins, cam16, width, height, want_uv=True):
    """rasterizer.py:93-202 — returns dict(triangle, texel, depth, u, v)."""
    v = _c(verts, np.float64).reshape(-1, 3)
    t = _c(tris, np.int32).reshape(-1, 3)
    s = _c(steps, np.int32)
    o = _c(origins, np.int8)
    cam = _c(cam16, np.float64)
    H, W = int(height), int(width)
    tri = np.empty((H, W), np.int32)
    tex = np.empty((H, W), np.int32)
    dep = np.empty((H, W), np.float64)
    u = np.empty((H, W), np.float64) if want_uv else None
    vv = np.empty((H, W), np.float64) if want_uv else None
    rc = lib().tfo_rasterize(_ptr(v), len(v), _ptr(t), len(t), _ptr(s), _ptr(o), _ptr(cam), W, H,
                             _ptr(tri), _ptr(tex), _ptr(dep), _ptr(u), _ptr(vv))
    if rc:
        raise MemoryError("oracle rasterize failed")
    return {"triangle": tri, "texel": tex, "depth": dep, "u": u, "v": vv}


def pixel_rows(offsets, tri, texel):
    """Global texel row per pixel (fusion.py:167, renderback.py:45); -1 where uncovered."""
    tri = np.asarray(tri)
    rows = np.full(tri.shape, -1, dtype=np.int64)
    cov = tri != -1
    rows[cov] = np.asarray(offsets, dtype=np.int64)[tri[cov]] + np.asarray(texel)[cov]
    return rows


def compute_pixel_weights(tri, texel, mode, alpha=None):
    """fusion.py:114-142."""
    if mode not in WEIGHT_MODES:
        raise ValueError("unknown weight mode %r" % (mode,))
    if mode == "blend" and (alpha is None or not 0.0 <= alpha <= 1.0):
        raise ValueError("blend weight mode needs alpha in [0, 1]")
    tri = np.asarray(tri)
    w = np.zeros(tri.shape, dtype=np.float64)
    cov = tri != -1
    if not cov.any():
        return w
    if mode == "pixels_iid":
        w[cov] = 1.0
        return w
    key = tri[cov].astype(np.int64) << 32 | np.asarray(texel)[cov].astype(np.int64)
    _, inverse, counts = np.unique(key, return_inverse=True, return_counts=True)
    per_image = 1.0 / counts[inverse]
    w[cov] = per_image if mode == "images_iid" else (1.0 - alpha) + alpha * per_image
    return w


def accumulate_frame(accum, counts, offsets, tri, texel, probs, weights, aggregator):
    """fusion.py:145-183 — folds one frame into float64 accum / int64 counts in place."""
    cov = np.asarray(tri) != -1
    if not cov.any():
        return
    rows = np.asarray(offsets, dtype=np.int64)[np.asarray(tri)[cov]] + np.asarray(texel)[cov]
    p = np.asarray(probs)[cov].astype(np.float64)
    w = np.asarray(weights)[cov].astype(np.float64)
    if aggregator == "sum":
        contrib = w[:, None] * p
    elif aggregator == "maxsum":
        keep = p == p.max(axis=1, keepdims=True)
        contrib = w[:, None] * np.where(keep, p, 0.0)
    elif aggregator == "mul":
        contrib = w[:, None] * np.log(np.clip(p, MUL_CLAMP, 1.0))
    else:
        raise ValueError("unknown aggregator %r" % (aggregator,))
    n = accum.shape[0]
    for k in range(accum.shape[1]):
        accum[:, k] += np.bincount(rows, weights=contrib[:, k], minlength=n)
    counts += np.bincount(rows, minlength=n)


def finalize(accum, counts, aggregator):
    """fusion.py:186-210 — returns (rows float32, unobserved bool)."""
    c = accum.shape[1]
    if aggregator == "mul":
        unobserved = counts == 0
        shifted = accum - accum.max(axis=1, keepdims=True)
        rows = np.exp(shifted)
        rows /= rows.sum(axis=1, keepdims=True)
    else:
        norm = accum.sum(axis=1)
        unobserved = (counts == 0) | (norm <= 0)
        safe = np.where(norm > 0, norm, 1.0)
        rows = accum / safe[:, None]
    rows[unobserved] = 1.0 / c
    return rows.astype(np.float32), unobserved


def texel_argmax(rows, unobserved):
    """fusion.py:213-222."""
    labels = rows.argmax(axis=1).astype(np.int32)
    labels[unobserved] = UNKNOWN
    return labels


def render_labels(texel_labels, offsets, tri, texel, fallback=None):
    """renderback.py:28-56."""
    tri = np.asarray(tri)
    out = np.full(tri.shape, UNKNOWN, dtype=np.int32)
    cov = tri != -1
    rows = np.asarray(offsets, dtype=np.int64)[tri[cov]] + np.asarray(texel)[cov]
    out[cov] = np.asarray(texel_labels)[rows]
    if fallback is not None:
        hole = out == UNKNOWN
        out[hole] = np.asarray(fallback)[hole]
    return out


def fuse_frames_c(verts, tris, steps, origins, offsets, n_x, cams, width, height, probs_list,
                  aggregator, weight_mode, alpha=0.0, accum=None, counts=None, nthreads=0):
    """Frame-parallel CPU fuse loop (rasterize → weights → accumulate, fusion.py:114-183)
    over OpenMP threads with private float64 accumulators; the CPU baseline."""
    v = _c(verts, np.float64).reshape(-1, 3)
    t = _c(tris, np.int32).reshape(-1, 3)
    s = _c(steps, np.int32)
    o = _c(origins, np.int8)
    off = _c(offsets, np.int64)
    cams = _c(cams, np.float64).reshape(-1, 16)
    c = int(probs_list[0].shape[-1])
    probs_list = [_c(p, np.float32) for p in probs_list]
    if accum is None:
        accum = np.zeros((n_x, c), np.float64)
    if counts is None:
        counts = np.zeros(n_x, np.int64)
    ptrs = (ctypes.c_void_p * len(probs_list))(*[p.ctypes.data for p in probs_list])
    agg = AGGREGATORS.index(aggregator)
    wm = WEIGHT_MODES.index(weight_mode)
    rc = lib().tfo_fuse_frames(_ptr(v), len(v), _ptr(t), len(t), _ptr(s), _ptr(o), _ptr(off), n_x, c,
                               _ptr(cams), int(width), int(height), len(probs_list),
                               ctypes.cast(ptrs, ctypes.c_void_p), agg, wm, float(alpha or 0.0),
                               _ptr(accum), _ptr(counts), int(nthreads))
    if rc:
        raise MemoryError("oracle fuse failed")
    return accum, counts


def worst_case_areas(verts, tris, cams, sizes):
    """geometry.py:360-380 (compute_worst_case_areas) via the C restatement."""
    v = _c(verts, np.float64).reshape(-1, 3)
    t = _c(tris, np.int32).reshape(-1, 3)
    cams = _c(cams, np.float64).reshape(-1, 16)
    sizes = _c(sizes, np.int32).reshape(-1, 2)
    areas = np.zeros(len(t), np.float64)
    lib().tfo_worst_case_areas(_ptr(v), len(v), _ptr(t), len(t), _ptr(cams), _ptr(sizes), len(cams), _ptr(areas))
    return areas


def build_steps(areas, gamma, max_steps=1024):
    """geometry.py:272-281 — per-triangle steps from areas."""
    areas = np.asarray(areas, dtype=np.float64)
    if gamma == 0:
        steps = np.ones(len(areas), dtype=np.int64)
    else:
        steps = np.maximum(1, np.ceil(gamma * np.sqrt(areas)).astype(np.int64))
    return np.minimum(steps, max_steps)


def finalize_c(accum, counts, aggregator, want_rows=True):
    n_x, c = accum.shape
    a = _c(accum, np.float64)
    cn = _c(counts, np.int64)
    rows = np.empty((n_x, c), np.float32) if want_rows else None
    unobs = np.empty(n_x, np.uint8)
    labels = np.empty(n_x, np.int32)
    lib().tfo_finalize(_ptr(a), _ptr(cn), n_x, c, AGGREGATORS.index(aggregator), _ptr(rows),
                       _ptr(unobs), _ptr(labels))
    return rows, unobs.astype(bool), labels

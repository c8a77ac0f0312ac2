"""In-process fusion sessions (texelfuse_bindings/__init__.py:1-141) on the GPU.

Public surface, names and error behaviour of the reference bindings:
``open_session`` / ``add_frame`` / ``finalize_and_render``.  A session keeps
mesh, layout and texture in device memory.  ``add_frame`` validates the frame,
takes its correspondence through the ``rasterize`` hook (lazy: no device work
yet) and queues the frame on the session's MeshAnnotation, which folds queued
frames as one batch (rasterization with fused hit counts, one scatter-add
launch that also writes each frame's network-argmax fallback) when the batch
is full or anything reads the texture.  It returns the covered-pixel count as
an int-like FrameCount resolved when read, so nothing synchronizes per
frame.
"""

import threading

import numpy as np
import torch

from .annotation import FallbackMap, MeshAnnotation
from .device import scene_for
from .errors import DataError
from .fusion import finalize, init_texture, parse_weight_mode
from .geometry import build_texel_layout, compute_worst_case_areas
from .meshio import load_mesh, load_trajectory

__all__ = ["open_session", "add_frame", "finalize_and_render"]


class _FusionSession:
    """Handle around (mesh, layout, texture, config) (bindings/__init__.py:38-65)."""

    def __init__(self, mesh, frames, layout, texture, weight_mode, alpha):
        self.mesh = mesh
        self.frames = {f.frame_id: f for f in frames}
        self.layout = layout
        self.texture = texture
        self.weight_mode = weight_mode
        self.alpha = alpha
        self.scene = scene_for(mesh, layout, texture.device)
        self.ann = MeshAnnotation(mesh, layout, weight_mode=_spec(weight_mode, alpha), texture=texture,
                                  device=texture.device)
        self.ann.fallbacks = FallbackMap()  # frame_id -> (H*W,) int32 device tensor (the frame's own argmax)
        sizes = {}
        for f in frames:
            sizes[(f.width, f.height)] = sizes.get((f.width, f.height), 0) + 1
        for size, n in sizes.items():  # one add per trajectory frame fits without allocating per batch
            self.ann.fallbacks.reserve(size, n)
        self._gate = threading.Lock()

    @property
    def fallbacks(self):
        return self.ann.fallbacks

    @property
    def num_texels(self):
        return int(self.layout.total_texels)

    @property
    def num_classes(self):
        return int(self.texture.num_classes)

    @property
    def finalized(self):
        return bool(self.texture.finalized)


def _spec(mode, alpha):
    return "blend:%r" % alpha if mode == "blend" else mode


def open_session(mesh_path, trajectory_path, gamma, aggregator, weight_mode, num_classes,
                 accum_dtype="fixed64", device=None):
    """Load the scene; size the texture from the worst-case projected footprints
    computed on the GPU (bindings/__init__.py:68-82).  The default fixed64
    accumulator makes a session's outputs independent of scheduling, so they
    equal the fuse command's in deterministic mode bit for bit (criterion 11)."""
    mesh = load_mesh(mesh_path)
    frames = load_trajectory(trajectory_path)
    mode, alpha = parse_weight_mode(weight_mode)
    areas = compute_worst_case_areas(mesh, frames)
    layout = build_texel_layout(mesh, areas, gamma)
    texture = init_texture(layout, num_classes, aggregator, accum_dtype=accum_dtype, device=device)
    return _FusionSession(mesh, frames, layout, texture, mode, alpha)


# module-level hook, as in the reference bindings (its tests monkeypatch bindings.rasterize)
from .rasterizer import rasterize  # noqa: E402


def add_frame(session, frame_id, probabilities):
    """Fold one frame's H x W x c probabilities; returns the pixel observations
    added (bindings/__init__.py:85-115)."""
    if not session._gate.acquire(blocking=False):
        raise RuntimeError("another add_frame call is running on this session")
    try:
        frame = session.frames.get(frame_id)
        if frame is None:
            raise DataError("frame %r is not in the trajectory (%d frames)" % (frame_id, len(session.frames)))
        want = (frame.height, frame.width, session.num_classes)
        shape = tuple(probabilities.shape) if hasattr(probabilities, "shape") else np.shape(probabilities)
        if shape != want:
            raise DataError("probability array shape %s does not match expected %s" % (shape, want))
        tex = session.texture
        if tex.finalized:
            raise RuntimeError("texture is already finalized")
        ids = rasterize(session.mesh, session.layout, frame)  # lazy IdImage: the fold rasterizes it
        return session.ann._enqueue(probabilities, frame, ids=ids, fallback_key=frame_id, want_count=True)
    finally:
        session._gate.release()


def finalize_and_render(session, frame_ids=()):
    """Finalize once, then label images for ``frame_ids`` (bindings/__init__.py:118-141).
    Returns rows, or (list of (H, W) int32 images, rows)."""
    frame_ids = list(frame_ids)
    missing = [fid for fid in frame_ids if fid not in session.frames]
    if missing:
        raise DataError("frame ids not in the trajectory: %s" % missing)
    tex = finalize(session.texture)
    rows = np.ascontiguousarray(tex.rows.copy())
    if not frame_ids:
        return rows
    # one batched rasterize + gather per frame size (renderback.py:28-56 with the
    # session's cached network argmax as fallback, bindings/__init__.py:136-141)
    images = [None] * len(frame_ids)
    by_size = {}
    for k, fid in enumerate(frame_ids):
        fr = session.frames[fid]
        by_size.setdefault((fr.width, fr.height), []).append(k)
    for (W, H), ks in by_size.items():
        frs = [session.frames[frame_ids[k]] for k in ks]
        fbs = [session.fallbacks.get(frame_ids[k]) for k in ks]
        fb = None
        if any(f is not None for f in fbs):
            fb = torch.stack([f if f is not None else torch.full((H * W,), -1, dtype=torch.int32,
                                                                 device=tex.device) for f in fbs])
        out = session.ann.render(frs, fallback=fb, host=True)
        for k, img in zip(ks, out):
            images[k] = np.ascontiguousarray(img)
    return images, rows

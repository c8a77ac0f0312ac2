"""In-process fusion sessions (texelfuse_bindings/__init__.py:1-141) on the GPU.

Public surface, names and error behaviour of the reference bindings:
``open_session`` / ``add_frame`` / ``finalize_and_render``.  A session keeps
mesh, layout and texture in device memory; ``add_frame`` runs the device
rasterizer, the fused scatter-add and the network-argmax fallback in one
pass and does not synchronize with the host: it returns a lazily evaluated
count of the pixel observations added.
"""

import threading

import numpy as np
import torch

from . import _native as N
from .device import scene_for
from .errors import DataError
from .fusion import finalize, init_texture, parse_weight_mode
from .geometry import build_texel_layout, compute_worst_case_areas
from .meshio import load_mesh, load_trajectory
from .renderback import render_labels_device

__all__ = ["open_session", "add_frame", "finalize_and_render"]


class LazyCount:
    """An int-like observation count that syncs with the device only when read."""

    __slots__ = ("_t", "_v")

    def __init__(self, tensor):
        self._t = tensor
        self._v = None

    def __int__(self):
        if self._v is None:
            self._v = int(self._t.item())
            self._t = None
        return self._v

    __index__ = __int__

    def __eq__(self, o):
        return int(self) == int(o)

    def __ne__(self, o):
        return int(self) != int(o)

    def __lt__(self, o):
        return int(self) < o

    def __le__(self, o):
        return int(self) <= o

    def __gt__(self, o):
        return int(self) > o

    def __ge__(self, o):
        return int(self) >= o

    def __hash__(self):
        return hash(int(self))

    def __add__(self, o):
        return int(self) + o

    __radd__ = __add__

    def __sub__(self, o):
        return int(self) - o

    def __rsub__(self, o):
        return o - int(self)

    def __repr__(self):
        return repr(int(self))


class _FusionSession:
    """Handle around (mesh, layout, texture, config) (bindings/__init__.py:38-65)."""

    def __init__(self, mesh, frames, layout, texture, weight_mode, alpha):
        self.mesh = mesh
        self.frames = {f.frame_id: f for f in frames}
        self.layout = layout
        self.texture = texture
        self.weight_mode = weight_mode
        self.alpha = alpha
        self.fallbacks = {}  # frame_id -> (H*W,) int32 device tensor (the frame's own argmax)
        self.scene = scene_for(mesh, layout, texture.device)
        self._gate = threading.Lock()

    @property
    def num_texels(self):
        return int(self.layout.total_texels)

    @property
    def num_classes(self):
        return int(self.texture.num_classes)

    @property
    def finalized(self):
        return bool(self.texture.finalized)


def open_session(mesh_path, trajectory_path, gamma, aggregator, weight_mode, num_classes,
                 accum_dtype="float64", device=None):
    """Load the scene; size the texture from the worst-case projected footprints
    computed on the GPU (bindings/__init__.py:68-82)."""
    mesh = load_mesh(mesh_path)
    frames = load_trajectory(trajectory_path)
    mode, alpha = parse_weight_mode(weight_mode)
    areas = compute_worst_case_areas(mesh, frames)
    layout = build_texel_layout(mesh, areas, gamma)
    texture = init_texture(layout, num_classes, aggregator, accum_dtype=accum_dtype, device=device)
    return _FusionSession(mesh, frames, layout, texture, mode, alpha)


def rasterize(mesh, layout, frame):
    """Module-level hook (the reference tests monkeypatch bindings.rasterize)."""
    from .rasterizer import rasterize as _r

    return _r(mesh, layout, frame)


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
        ids = rasterize(session.mesh, session.layout, frame)
        scene = session.scene
        H, W, c = want
        hw = H * W
        if isinstance(probabilities, torch.Tensor):
            p = probabilities.detach().to(device=tex.device, dtype=torch.float32).contiguous()
        else:
            p = torch.as_tensor(np.ascontiguousarray(probabilities, dtype=np.float32)).to(tex.device)
        if p.data_ptr() % 16:
            p = p.clone()
        rows = ids.rows_on(scene)
        tex._push_host()
        hits = None
        if session.weight_mode != "pixels_iid":
            hits = scene.hits(1)
            N.call("tfb_count_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle())
        fb = torch.empty(hw, dtype=torch.int32, device=tex.device)
        parr, _keep = N.ptr_array([p.data_ptr()])
        N.call("tfb_fuse", N.ptr(rows), hw, 1, parr, c, N.ptr(hits), None, tex.total_texels,
               N.AGG_IDS[tex.aggregator], N.WMODE_IDS[session.weight_mode], float(session.alpha or 0.0),
               N.ptr(tex._accum), int(tex.is_f64), tex.stride, N.ptr(tex._counts), N.ptr(fb), N.stream_handle())
        if hits is not None:
            N.call("tfb_clear_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle())
        tex._h_accum = tex._h_counts = None
        session.fallbacks[frame_id] = fb
        return LazyCount((rows >= 0).sum())
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
    labels = tex.labels_device
    rows = np.ascontiguousarray(tex.rows.copy())
    if not frame_ids:
        return rows
    images = []
    for fid in frame_ids:
        fr = session.frames[fid]
        ids = rasterize(session.mesh, session.layout, fr)
        hw = fr.width * fr.height
        out = render_labels_device(labels, ids.rows_on(session.scene), hw, 1, session.fallbacks.get(fid))
        images.append(out.view(fr.height, fr.width).cpu().numpy())
    return images, rows

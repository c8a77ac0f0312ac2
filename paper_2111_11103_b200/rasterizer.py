"""Per-frame correspondences (rasterizer.py:93-202) on the GPU.

``rasterize`` returns an IdImage that is lazy: it records the camera, and the
frame is rasterized on the device when something needs its planes (the row
image for fusion or render, or a host view).  A session / MeshAnnotation that
receives such an IdImage rasterizes it inside its batched fold instead, with
the texel hit counts fused in.  The host views ``triangle``/``texel``/
``depth``/``u``/``v`` are materialized on first access (depth/u/v by a
second, bit-identical rasterization that also writes those float64 planes —
only tests and debugging read them).
IdImages can also be built on the host from arrays, as the reference's test
helpers do (tests/helpers.py:45-61); they are uploaded when first used.
"""

import numpy as np
import torch

from . import _native as N
from .device import scene_for
from .errors import DataError
from .geometry import pack_camera

DEPTH_TIE = 1e-9  # rasterizer.py:18
NONE = -1  # rasterizer.py:20


class IdImage:
    """Per-pixel (triangle, texel) correspondence of one frame (rasterizer.py:23-43)."""

    def __init__(self, frame_id, width, height, triangle=None, texel=None, depth=None, u=None, v=None):
        self.frame_id = frame_id
        self.width = int(width)
        self.height = int(height)
        self._host = {}
        for name, arr in (("triangle", triangle), ("texel", texel), ("depth", depth), ("u", u), ("v", v)):
            if arr is not None:
                if isinstance(arr, torch.Tensor):
                    arr = arr.detach().cpu().numpy()
                self._host[name] = np.asarray(arr)
        self._rows = None  # (H*W,) int32 device rows for _rows_scene
        self._rows_scene = None
        self._dev_tri = None
        self._dev_texel = None
        self._source = None  # (scene, camera record) for lazily re-rendered planes

    # -- construction from the device path -------------------------------------
    @classmethod
    def _from_camera(cls, frame_id, width, height, scene, cam):
        """Lazy IdImage of ``scene`` seen from the packed camera ``cam`` ((16,) float64)."""
        ids = cls(frame_id, width, height)
        ids._source = (scene, np.asarray(cam, dtype=np.float64).reshape(16))
        return ids

    def _cam_device(self):
        scene, cam = self._source
        return torch.as_tensor(cam.reshape(1, 16)).to(scene.device, non_blocking=True)

    def _ensure_device(self):
        """Rasterize a lazy IdImage once: row image + triangle / texel planes."""
        if self._rows is not None or self._source is None:
            return
        scene, _cam = self._source
        hw = self.width * self.height
        d = scene.device
        rows = torch.empty((1, hw), dtype=torch.int32, device=d)
        tri = torch.empty((1, hw), dtype=torch.int32, device=d)
        tex = torch.empty((1, hw), dtype=torch.int32, device=d)
        with torch.cuda.device(d):
            scene.rasterize(self._cam_device(), self.width, self.height, rows, tri=tri, texel=tex)
        self._rows, self._rows_scene = rows.view(-1), scene
        self._dev_tri, self._dev_texel = tri.view(-1), tex.view(-1)

    # -- reference field access ---------------------------------------------------
    def _materialize(self, name):
        if name in self._host:
            return self._host[name]
        H, W = self.height, self.width
        if name in ("triangle", "texel"):
            self._ensure_device()
        if name in ("triangle", "texel") and self._dev_tri is not None:
            self._host["triangle"] = N.host_copy(self._dev_tri.view(H, W))
            self._host["texel"] = N.host_copy(self._dev_texel.view(H, W))
            return self._host[name]
        if self._source is None:
            raise AttributeError("IdImage has no %s plane" % name)
        scene, _cam = self._source
        cam = self._cam_device()
        d = scene.device
        rows = torch.empty((1, H * W), dtype=torch.int32, device=d)
        tri = torch.empty((1, H * W), dtype=torch.int32, device=d)
        tex = torch.empty((1, H * W), dtype=torch.int32, device=d)
        dep = torch.empty((1, H * W), dtype=torch.float64, device=d)
        uu = torch.empty((1, H * W), dtype=torch.float64, device=d)
        vv = torch.empty((1, H * W), dtype=torch.float64, device=d)
        with torch.cuda.device(d):
            scene.rasterize(cam, W, H, rows, tri=tri, texel=tex, depth=dep, u=uu, v=vv)
        for key, t in (("triangle", tri), ("texel", tex), ("depth", dep), ("u", uu), ("v", vv)):
            self._host.setdefault(key, N.host_copy(t.view(H, W)))
        return self._host[name]

    triangle = property(lambda self: self._materialize("triangle"))
    texel = property(lambda self: self._materialize("texel"))
    depth = property(lambda self: self._materialize("depth"))
    u = property(lambda self: self._materialize("u"))
    v = property(lambda self: self._materialize("v"))

    @property
    def covered(self):
        return self.triangle != NONE

    # -- device rows ----------------------------------------------------------------
    def rows_on(self, scene):
        """(H*W,) int32 device tensor of global texel rows (offsets[t] + texel, -1 uncovered)."""
        if self._source is not None and not self._host:
            self._ensure_device()
        if self._rows is not None and self._rows_scene is not None and (
                self._rows_scene is scene or self._rows_scene.same_layout(scene.layout)):
            return self._rows
        tri = np.ascontiguousarray(self.triangle, dtype=np.int32).reshape(-1)
        tex = np.ascontiguousarray(self.texel, dtype=np.int32).reshape(-1)
        if tri.size != self.width * self.height:
            raise DataError("IdImage planes do not match its %dx%d size" % (self.width, self.height))
        d = scene.device
        t_tri = torch.as_tensor(tri).to(d)
        t_tex = torch.as_tensor(tex).to(d)
        rows = torch.empty(tri.size, dtype=torch.int32, device=d)
        bad = torch.zeros(1, dtype=torch.int32, device=d)
        N.call("tfb_rows_from_ids", N.ptr(t_tri), N.ptr(t_tex), tri.size, scene.sref, N.ptr(rows), N.ptr(bad),
               N.stream_handle())
        if int(bad.item()):
            raise DataError("IdImage references triangles or texels outside the layout")
        self._rows, self._rows_scene = rows, scene
        return rows


def rasterize(mesh, layout, frame, device=None):
    """Render triangle/texel correspondences for one frame (rasterizer.py:93-132).
    Lazy: the device rasterization runs when the IdImage is first used."""
    if layout.num_triangles != mesh.num_triangles:
        raise DataError("layout covers %d triangles but mesh has %d" % (layout.num_triangles, mesh.num_triangles))
    scene = scene_for(mesh, layout, device)
    return IdImage._from_camera(frame.frame_id, int(frame.width), int(frame.height), scene, pack_camera(frame))


def project_point(frame, point):
    """Project one world point → (x_px, y_px, depth) (rasterizer.py:46-59)."""
    p = np.asarray(point, dtype=np.float64).reshape(1, 3) @ frame.rotation.T + frame.translation
    z = float(p[0, 2])
    if z == 0.0:
        return float("nan"), float("nan"), 0.0
    return float(p[0, 0] / z * frame.fx + frame.cx), float(p[0, 1] / z * frame.fy + frame.cy), z


def pixel_world_points(mesh, layout, ids):
    """World position of every covered pixel from its (u, v) (rasterizer.py:205-224)."""
    cov = ids.covered
    tri = ids.triangle[cov].astype(np.int64)
    u, v = ids.u[cov], ids.v[cov]
    o = layout.origins[tri].astype(np.int64)
    w = np.empty((len(tri), 3))
    r = np.arange(len(tri))
    w[r, o] = 1.0 - u
    w[r, (o + 1) % 3] = u - v
    w[r, (o + 2) % 3] = v
    return np.einsum("nk,nkd->nd", w, mesh.vertices[mesh.triangles[tri]])


def dump_debug_images(ids, prefix):
    """16-bit grayscale PNGs of an IdImage for eyeballing correspondences
    (rasterizer.py:227-254): hashed triangle id, texel id + 1 and depth
    rescaled to [1, 65535]; 0 marks uncovered pixels.  Returns the paths."""
    from PIL import Image

    cov = ids.covered
    tri = ids.triangle.astype(np.int64)
    planes = {
        "triangle": np.where(cov, (tri + 1) * 2654435761 % 65535 + 1, 0),
        "texel": np.where(cov, ids.texel.astype(np.int64) % 65535 + 1, 0),
        "depth": np.zeros(cov.shape, np.int64),
    }
    if cov.any():
        d = ids.depth[cov]
        lo, hi = float(d.min()), float(d.max())
        planes["depth"][cov] = ((d - lo) * (65534.0 / (hi - lo) if hi > lo else 0.0)).astype(np.int64) + 1
    paths = []
    for name in ("triangle", "texel", "depth"):
        path = "%s_%s.png" % (prefix, name)
        img = planes[name].astype("<u2")
        Image.frombytes("I;16", (img.shape[1], img.shape[0]), img.tobytes()).save(path)
        paths.append(path)
    return paths

"""Device residency of the mesh + texel layout, and thin launch wrappers.

A DeviceScene holds the float64 vertices, int32 triangles and the layout
arrays in HBM (uploaded once) plus per-(width, height, batch) scratch, and
launches the C-ABI kernels on the caller's CUDA stream.  All buffers are
torch tensors (PyTorch is the allocator); the library never allocates.
"""

import ctypes
import os

import numpy as np
import torch

from . import _native as N
from .geometry import pack_camera

_CACHE_ATTR = "_tfb_device_scene"


CLUSTER = 64     # triangle slots per cluster (tfb_cluster.tri)
CLUSTER_V = 128  # vertex slots per cluster (tfb_cluster.verts)

# numpy mirror of tfb_cluster (include/texelfuse_b200.h), 1856 bytes
CLUSTER_DTYPE = np.dtype([("tri", "<i4", (CLUSTER, 4)), ("local", "<u4", (CLUSTER,)), ("nverts", "<i4"),
                          ("pad", "<i4", (3,)), ("verts", "<i4", (CLUSTER_V,)), ("box", "<f8", (6,))])
assert CLUSTER_DTYPE.itemsize == 1856


def _spread10(x):
    """Interleave the low 10 bits of x with two zero bits (3-D Morton code)."""
    x = x & np.uint64(0x3FF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x030000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x0300F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x030C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x09249249)
    return x


def build_clusters(vertices, triangles):
    """Spatial clusters of a mesh for tfb_scene.clusters: triangles in Morton
    order of their centroids, 64 consecutive ones per cluster (32 where 64 would
    use more than 128 distinct vertices), each cluster's distinct vertices with
    the corners' local indices, and the world AABB of those vertices.  Returns a
    structured array of CLUSTER_DTYPE."""
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles, dtype=np.int64)
    m, nv = len(t), len(v)
    if m == 0:
        return np.zeros(0, dtype=CLUSTER_DTYPE)
    cent = v[t].mean(axis=1)
    lo, hi = cent.min(axis=0), cent.max(axis=0)
    span = np.where(hi > lo, hi - lo, 1.0)
    q = np.clip(((cent - lo) / span * 1023.0), 0, 1023).astype(np.uint64)
    code = _spread10(q[:, 0]) | (_spread10(q[:, 1]) << np.uint64(1)) | (_spread10(q[:, 2]) << np.uint64(2))
    order = np.argsort(code, kind="stable")

    def distinct_per_segment(starts, lens):
        seg = np.repeat(np.arange(len(starts)), lens)
        pos = np.arange(m)  # the segments tile the Morton order contiguously
        corners = t[order[pos]]                                   # (n, 3)
        keys = seg[:, None].astype(np.int64) * nv + corners       # distinct per segment
        uk, inv = np.unique(keys.ravel(), return_inverse=True)
        useg = uk // nv
        first = np.searchsorted(useg, np.arange(len(starts)))
        counts = np.bincount(useg, minlength=len(starts))
        return seg, pos, corners, uk % nv, useg, first, counts, inv.reshape(-1, 3)

    starts = np.arange(0, m, CLUSTER)
    lens = np.minimum(CLUSTER, m - starts)
    res = distinct_per_segment(starts, lens)
    big = res[6] > CLUSTER_V
    if big.any():  # halves of 32 triangles use at most 96 distinct vertices
        s2, l2 = [], []
        for s0, n, b in zip(starts, lens, big):
            if b:
                s2 += [s0, s0 + n // 2]
                l2 += [n // 2, n - n // 2]
            else:
                s2.append(s0)
                l2.append(n)
        starts, lens = np.array(s2), np.array(l2)
        res = distinct_per_segment(starts, lens)
    seg, pos, corners, uvid, useg, first, counts, inv = res
    nc = len(starts)
    out = np.zeros(nc, dtype=CLUSTER_DTYPE)
    slot = pos - np.repeat(starts, lens)
    tri = np.full((nc, CLUSTER, 4), 0, dtype=np.int32)
    tri[:, :, 0] = -1
    tri[seg, slot, 0] = order[pos]
    tri[seg, slot, 1:] = corners
    out["tri"] = tri
    local = inv - first[seg][:, None]
    loc = np.zeros((nc, CLUSTER), dtype=np.uint32)
    loc[seg, slot] = (local[:, 0] | (local[:, 1] << 8) | (local[:, 2] << 16)).astype(np.uint32)
    out["local"] = loc
    out["nverts"] = counts
    vslot = np.arange(len(uvid)) - first[useg]
    verts = np.zeros((nc, CLUSTER_V), dtype=np.int32)
    verts[useg, vslot] = uvid
    out["verts"] = verts
    pv = v[uvid]  # grouped by cluster (uvid is sorted by cluster first)
    out["box"] = np.concatenate([np.minimum.reduceat(pv, first, axis=0), np.maximum.reduceat(pv, first, axis=0)],
                                axis=1)
    return out


def _dev(device):
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


class DeviceScene:
    """Mesh + layout in device memory (geometry.py:31-77, 208-232)."""

    def __init__(self, mesh, layout, device=None):
        """``mesh`` may be None for a layout-only scene (texel rows and fusion,
        no rasterization)."""
        N.require_cuda()
        if mesh is not None and layout.num_triangles != mesh.num_triangles:
            from .errors import DataError

            raise DataError("layout covers %d triangles but mesh has %d" % (layout.num_triangles, mesh.num_triangles))
        self.device = _dev(device)
        self.mesh = mesh
        self.layout = layout
        d = self.device
        verts = mesh.vertices if mesh is not None else np.zeros((0, 3))
        tris = mesh.triangles if mesh is not None else np.zeros((0, 3), np.int32)
        self.vertices = torch.as_tensor(np.ascontiguousarray(verts, np.float64), device=d)
        self.triangles = torch.as_tensor(np.ascontiguousarray(tris, np.int32), device=d)
        self.steps = torch.as_tensor(np.ascontiguousarray(layout.steps, np.int32), device=d)
        self.origins = torch.as_tensor(np.ascontiguousarray(layout.origins, np.int8), device=d)
        self.offsets = torch.as_tensor(np.ascontiguousarray(layout.offsets, np.int64), device=d)
        self.num_triangles = int(layout.num_triangles)
        self.total_texels = int(layout.total_texels)
        # spatial clusters for the rasterizer's cluster cull (results are identical
        # without them; TFB_NO_CLUSTERS=1 disables them)
        self.clusters = None
        nclusters = 0
        if mesh is not None and len(tris) > 0 and os.environ.get("TFB_NO_CLUSTERS", "0") != "1":
            cl = build_clusters(verts, tris)
            self.clusters = torch.as_tensor(cl.view(np.uint8), device=d)
            nclusters = len(cl)
        self.struct = N.TfbScene(
            self.vertices.data_ptr(), self.triangles.data_ptr(), self.steps.data_ptr(), self.origins.data_ptr(),
            self.offsets.data_ptr(), len(verts), self.num_triangles, self.total_texels,
            self.clusters.data_ptr() if nclusters else None, nclusters)
        self._sig = _signature(mesh, layout)
        self._ws = {}
        self._bufs = {}

    def matches(self, mesh, layout):
        return self._sig == _signature(mesh, layout)

    def same_layout(self, layout):
        return self.layout is layout or self._sig[4:] == _signature(None, layout)[4:]

    @property
    def sref(self):
        return ctypes.byref(self.struct)

    # -- scratch ---------------------------------------------------------------
    def workspace(self, width, height, nframes):
        key = (width, height)
        ws = self._ws.get(key)
        if ws is None or ws[0] < nframes:
            nbytes = N.load().tfb_raster_workspace_bytes(int(self.struct.num_vertices), self.num_triangles, width,
                                                         height, nframes, 0)
            ws = (nframes, torch.empty(nbytes, dtype=torch.uint8, device=self.device))
            self._ws[key] = ws
        return ws[1]

    def buffer(self, name, shape, dtype, zero=False):
        """Named persistent scratch (grown on demand, never shrunk)."""
        n = int(np.prod(shape))
        t = self._bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = (torch.zeros if zero else torch.empty)(max(n, 1), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[:n].view(*shape)

    def hits(self, nframes):
        """Per-frame texel hit counters; kept all-zero between uses by tfb_clear_hits."""
        return self.buffer("hits", (nframes, max(self.total_texels, 1)), torch.int32, zero=True)

    # -- launches --------------------------------------------------------------
    def rasterize(self, cams, width, height, rows, hits=None, tri=None, texel=None, depth=None, u=None, v=None,
                  stream=None, phases=3):
        """cams: (B, 16) float64 device tensor; rows: (B, H*W) int32 device tensor.
        phases: 1 = cull + setup + binning, 2 = the tile kernels, 3 = both
        (tfb_rasterize_phases; the two halves of one batch take the same arguments)."""
        B = int(cams.shape[0])
        if B == 0:
            return
        if self.mesh is None:
            raise RuntimeError("layout-only scene cannot rasterize")
        ws = self.workspace(width, height, B)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):  # launches go to this scene's GPU, whatever is current
            N.call("tfb_rasterize_phases", self.sref, N.ptr(cams), B, int(width), int(height), N.ptr(ws),
                   ws.numel(), 0, N.ptr(rows), N.ptr(hits), N.ptr(tri), N.ptr(texel), N.ptr(depth), N.ptr(u),
                   N.ptr(v), int(phases), N.stream_handle(stream))

    def cams_tensor(self, frames):
        arr = np.stack([pack_camera(f) for f in frames]) if frames else np.zeros((0, 16))
        return torch.as_tensor(arr, dtype=torch.float64).to(self.device, non_blocking=False)


def _signature(mesh, layout):
    mv = (id(mesh.vertices), id(mesh.triangles), mesh.vertices.shape, mesh.triangles.shape) if mesh is not None \
        else (None, None, None, None)
    return mv + (id(layout.steps), id(layout.origins), id(layout.offsets), int(layout.total_texels))


def scene_for(mesh, layout, device=None):
    """Cached DeviceScene for (mesh, layout), keyed on array identity."""
    cached = getattr(layout, _CACHE_ATTR, None)
    if cached is not None and cached.matches(mesh, layout) and (device is None or cached.device == _dev(device)):
        return cached
    sc = DeviceScene(mesh, layout, device)
    try:
        object.__setattr__(layout, _CACHE_ATTR, sc)
    except Exception:  # pragma: no cover
        pass
    return sc


def layout_scene(layout, device=None):
    """Cached layout-only DeviceScene (offsets/steps for fusion of host IdImages)."""
    cached = getattr(layout, "_tfb_layout_scene", None)
    if cached is not None and cached.same_layout(layout) and (device is None or cached.device == _dev(device)):
        return cached
    full = getattr(layout, _CACHE_ATTR, None)
    if full is not None and full.same_layout(layout) and (device is None or full.device == _dev(device)):
        return full
    sc = DeviceScene(None, layout, device)
    object.__setattr__(layout, "_tfb_layout_scene", sc)
    return sc


class _MeshOnly:
    """Layout stand-in for kernels that only read the mesh (area pass)."""

    def __init__(self, m):
        self.steps = np.ones(m, np.int32)
        self.origins = np.zeros(m, np.int8)
        self.offsets = np.arange(m, dtype=np.int64)
        self.total_texels = m
        self.num_triangles = m


def worst_case_areas(mesh, frames, device=None):
    """compute_worst_case_areas (geometry.py:360-380) on the GPU; returns host float64 (m,)."""
    N.require_cuda()
    sc = DeviceScene(mesh, _MeshOnly(mesh.num_triangles), device)
    cams = sc.cams_tensor(frames)
    sizes = torch.as_tensor(np.array([[f.width, f.height] for f in frames], dtype=np.int32)).to(sc.device)
    areas = torch.zeros(mesh.num_triangles, dtype=torch.float64, device=sc.device)
    N.call("tfb_worst_case_areas", sc.sref, N.ptr(cams), N.ptr(sizes), len(frames), N.ptr(areas),
           N.stream_handle())
    return areas.cpu().numpy()

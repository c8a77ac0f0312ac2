"""Host-side data model: mesh, pinhole cameras and the texel layout.

Semantics follow the reference geometry module (texelfuse/geometry.py); the
classes are plain host containers that the device code reads once.  The
texel parametrization (geometry.py:1-10): a triangle with ``s`` steps has
``(s*s + s)/2`` texels; the texel at cell (i, j), 0 <= j <= i < s, has
packed id ``(i*i + i)/2 + j``.  ``offsets[t] + id`` is the global row.
"""

import logging
from dataclasses import dataclass

import numpy as np

from .errors import DataError

log = logging.getLogger("texelfuse.geometry")

DEGENERATE_AREA = 1e-12  # geometry.py:24
NEAR_PLANE = 1e-4  # geometry.py:26
MAX_STEPS = 1024  # geometry.py:28


def _tri_areas(vertices, triangles):
    a = vertices[triangles[:, 0]]
    e1 = vertices[triangles[:, 1]] - a
    e2 = vertices[triangles[:, 2]] - a
    return 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)


@dataclass(eq=False)
class Mesh:
    """World-space vertices (n, 3) float64 and triangles (m, 3) int32 (geometry.py:31-77)."""

    vertices: np.ndarray
    triangles: np.ndarray
    dropped_degenerate: int = 0

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int32).reshape(-1, 3)
        if self.triangles.size:
            lo, hi = int(self.triangles.min()), int(self.triangles.max())
            if lo < 0:
                raise DataError("negative vertex index in triangle list")
            if hi >= len(self.vertices):
                raise DataError("triangle references vertex %d but mesh has %d vertices" % (hi, len(self.vertices)))

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_triangles(self):
        return len(self.triangles)

    @classmethod
    def from_arrays(cls, vertices, triangles):
        """Build a mesh, dropping triangles whose 3D area is <= 1e-12 m^2."""
        v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.asarray(triangles, dtype=np.int32).reshape(-1, 3)
        dropped = 0
        if len(t):
            keep = _tri_areas(v, t) > DEGENERATE_AREA
            dropped = int(len(t) - keep.sum())
            if dropped:
                log.info("dropping %d degenerate triangles", dropped)
                t = t[keep]
        return cls(vertices=v, triangles=t, dropped_degenerate=dropped)


def triangle_areas(mesh):
    return _tri_areas(mesh.vertices, mesh.triangles)


@dataclass(frozen=True)
class Intrinsics:
    """Pinhole intrinsics; pixel centres at half-integer coordinates (geometry.py:92-107)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if not (self.fx > 0 and self.fy > 0):
            raise DataError("focal lengths must be positive")
        if not (self.width > 0 and self.height > 0):
            raise DataError("image dimensions must be positive")


@dataclass(eq=False)
class CameraFrame:
    """Posed camera: x_cam = R @ x_world + t, x right / y down / z forward (geometry.py:110-156)."""

    frame_id: int
    intrinsics: Intrinsics
    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        dev = float(np.abs(self.rotation @ self.rotation.T - np.eye(3)).max())
        if dev > 1e-6:
            raise DataError("frame %d: rotation is not orthonormal (max deviation %.3g)" % (self.frame_id, dev))

    fx = property(lambda self: self.intrinsics.fx)
    fy = property(lambda self: self.intrinsics.fy)
    cx = property(lambda self: self.intrinsics.cx)
    cy = property(lambda self: self.intrinsics.cy)
    width = property(lambda self: self.intrinsics.width)
    height = property(lambda self: self.intrinsics.height)

    def packed(self):
        """The 16-float64 camera record of the C ABI: R (row-major), t, fx, fy, cx, cy."""
        return pack_camera(self)


def pack_camera(frame):
    """The 16-float64 camera record of the C ABI: R (row-major), t, fx, fy, cx, cy."""
    i = frame.intrinsics
    return np.concatenate((np.asarray(frame.rotation, dtype=np.float64).reshape(9),
                           np.asarray(frame.translation, dtype=np.float64).reshape(3),
                           np.array((i.fx, i.fy, i.cx, i.cy), dtype=np.float64)))


def to_camera(frame, points):
    """World → camera coordinates of (n, 3) points (geometry.py:159-161)."""
    return np.asarray(points, dtype=np.float64) @ frame.rotation.T + frame.translation


def project_camera_points(frame, cam_points):
    """(x, y, depth) pixel projection of camera-space points (geometry.py:164-174)."""
    z = cam_points[..., 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        x = cam_points[..., 0] / z * frame.fx + frame.cx
        y = cam_points[..., 1] / z * frame.fy + frame.cy
    return x, y, z


def texel_count(steps):
    """(s*s + s)/2 texels per triangle (geometry.py:181-185)."""
    s = np.asarray(steps, dtype=np.int64)
    n = (s * s + s) // 2
    return n if n.ndim else int(n)


def texel_id(s, u, v):
    """Packed id of the texel holding (u, v), 0 <= v <= u < 1 (geometry.py:188-199)."""
    assert s >= 1, "subdivision steps must be >= 1"
    assert 0.0 <= v <= u < 1.0, "texel coordinates must satisfy 0 <= v <= u < 1"
    i, j = int(s * u), int(s * v)
    return (i * i + i) // 2 + j


def texel_ids_grid(s, i, j):
    i = np.asarray(i, dtype=np.int64)
    return (i * i + i) // 2 + np.asarray(j, dtype=np.int64)


@dataclass(eq=False)
class TexelLayout:
    """Per-triangle steps (int32), uv origins (int8), packed offsets (int64) (geometry.py:208-232)."""

    steps: np.ndarray
    origins: np.ndarray
    offsets: np.ndarray
    total_texels: int

    def __post_init__(self):
        self.steps = np.asarray(self.steps, dtype=np.int32)
        self.origins = np.asarray(self.origins, dtype=np.int8)
        self.offsets = np.asarray(self.offsets, dtype=np.int64)
        self.total_texels = int(self.total_texels)

    @property
    def num_triangles(self):
        return len(self.steps)

    def texel_counts(self):
        return texel_count(self.steps)


def uv_origins(vertices, triangles):
    """Vertex whose interior angle is nearest 90 degrees, ties to the lowest index
    (geometry.py:235-254)."""
    triangles = np.asarray(triangles)
    m = len(triangles)
    if m == 0:
        return np.zeros(0, dtype=np.int8)
    corners = [np.asarray(vertices)[triangles[:, k]] for k in range(3)]
    dev = np.empty((m, 3))
    for k in range(3):
        e1 = corners[(k + 1) % 3] - corners[k]
        e2 = corners[(k + 2) % 3] - corners[k]
        cosang = np.einsum("ij,ij->i", e1, e2)
        cosang /= np.linalg.norm(e1, axis=1) * np.linalg.norm(e2, axis=1)
        dev[:, k] = np.abs(np.arccos(np.clip(cosang, -1.0, 1.0)) - 0.5 * np.pi)
    return np.argmin(dev, axis=1).astype(np.int8)


def _packed(steps):
    counts = texel_count(steps)
    offsets = np.zeros(len(steps), dtype=np.int64)
    if len(steps):
        np.cumsum(counts[:-1], out=offsets[1:])
    return offsets, int(np.sum(counts))


def build_texel_layout(mesh, areas, gamma):
    """steps = max(1, ceil(gamma*sqrt(area))) clamped to MAX_STEPS (geometry.py:257-291)."""
    if gamma < 0:
        raise ValueError("gamma must be >= 0")
    areas = np.asarray(areas, dtype=np.float64)
    if areas.shape != (mesh.num_triangles,):
        raise DataError("areas shape %s does not match triangle count %d" % (areas.shape, mesh.num_triangles))
    if gamma == 0:
        steps = np.ones(mesh.num_triangles, dtype=np.int64)
    else:
        steps = np.maximum(1, np.ceil(gamma * np.sqrt(areas)).astype(np.int64))
    n_clamped = int(np.count_nonzero(steps > MAX_STEPS))
    if n_clamped:
        log.warning("clamping subdivision steps of %d triangles to %d", n_clamped, MAX_STEPS)
        steps = np.minimum(steps, MAX_STEPS)
    offsets, total = _packed(steps)
    return TexelLayout(steps=steps, origins=uv_origins(mesh.vertices, mesh.triangles), offsets=offsets,
                       total_texels=total)


def uniform_layout(mesh, steps=1):
    """Same subdivision for every triangle (geometry.py:294-305)."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    s = np.full(mesh.num_triangles, steps, dtype=np.int32)
    offsets, total = _packed(s)
    return TexelLayout(steps=s, origins=uv_origins(mesh.vertices, mesh.triangles), offsets=offsets,
                       total_texels=total)


def compute_worst_case_areas(mesh, frames):
    """Max projected pixel area per triangle over all frames (geometry.py:360-380), on the GPU."""
    from .device import worst_case_areas

    frames = list(frames)
    if not frames:
        raise ValueError("at least one frame is required")
    return worst_case_areas(mesh, frames)


__all__ = [
    "DEGENERATE_AREA", "NEAR_PLANE", "MAX_STEPS", "Mesh", "Intrinsics", "CameraFrame", "TexelLayout",
    "triangle_areas", "to_camera", "project_camera_points", "texel_count", "texel_id", "texel_ids_grid",
    "uv_origins", "build_texel_layout", "uniform_layout", "compute_worst_case_areas", "pack_camera",
]

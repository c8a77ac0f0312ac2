"""Synthetic scenes with exact ground truth: the fixture source of the
reference's tests and of ``texelfuse synth`` (texelfuse/synthgen.py), with
the same API so those tests run against this package unmodified.

Scene families: ``cube`` (one class per face), ``room`` (inward box, one
class per wall, the BASELINE mesh) and ``checker_sphere`` (a positional
checker finer than the triangles, so labels change inside faces).  Meshes,
trajectories and the Philox-keyed noise are bit-identical to the
reference's (synth.py); ground truth comes from this package's GPU
rasterizer, which is bit-exact with the reference's.  Not on the hot path.
"""

import os
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, DataError
from .formats import write_probability_image
from .fusion import UNKNOWN
from .geometry import Mesh, uniform_layout
from .meshio import save_ply, save_trajectory
from .rasterizer import pixel_world_points, rasterize
from .renderback import default_palette, save_palette, write_label_png
from . import synth as _s
from .synth import corrupt, look_at, make_icosphere, make_orbit_trajectory  # noqa: F401  (reference names)

SCENE_KINDS = ("cube", "room", "checker_sphere")
NOISE_KINDS = ("flip", "dirichlet")


@dataclass
class NoiseModel(_s.NoiseModel):
    """flip / dirichlet prediction noise with the reference's argument checks
    (synthgen.py:32-56)."""

    def __post_init__(self):
        if self.kind not in NOISE_KINDS:
            raise ConfigError("unknown noise kind %r (choose from %s)" % (self.kind, NOISE_KINDS))
        if not 0.0 <= self.epsilon < 1.0:
            raise ConfigError("epsilon must be in [0, 1)")
        if not 0.0 < self.q <= 1.0:
            raise ConfigError("q must be in (0, 1]")
        if self.kappa <= 0.0:
            raise ConfigError("kappa must be positive")


@dataclass
class SyntheticScene:
    """A mesh with its exact labels: per face, or a function of the surface point."""

    name: str
    mesh: Mesh
    num_classes: int
    face_labels: np.ndarray = None
    label_fn: object = None
    class_names: list = field(default_factory=list)

    def __post_init__(self):
        if (self.face_labels is None) == (self.label_fn is None):
            raise ValueError("scene needs exactly one of face_labels / label_fn")
        if self.face_labels is not None:
            self.face_labels = np.asarray(self.face_labels, dtype=np.int32)
            if self.face_labels.shape != (self.mesh.num_triangles,):
                raise DataError("face_labels do not match triangle count")


_CUBE_NAMES = ["x_plus", "x_minus", "y_plus", "y_minus", "z_plus", "z_minus"]
_ROOM_NAMES = ["floor", "ceiling", "wall_x_plus", "wall_x_minus", "wall_y_plus", "wall_y_minus"]


def make_cube(size=2.0, num_classes=6):
    """12-triangle cube; the two triangles of face k carry class k % num_classes."""
    if num_classes < 2:
        raise ConfigError("cube needs at least 2 classes")
    mesh = _s.make_cube(size)
    labels = np.repeat(np.arange(6) % num_classes, 2).astype(np.int32)
    return SyntheticScene("cube", mesh, num_classes, face_labels=labels,
                          class_names=_CUBE_NAMES[:num_classes] if num_classes <= 6 else [])


def make_room(size=(6.0, 5.0, 3.0), tess=4, num_classes=6):
    """Inward box, 2*tess^2 triangles per wall in the order floor, ceiling, +x, -x, +y, -y."""
    if num_classes < 2:
        raise ConfigError("room needs at least 2 classes")
    v, t = _s.make_room(size, tess)
    mesh = Mesh.from_arrays(v, t)
    labels = np.repeat(np.arange(6) % num_classes, 2 * tess * tess).astype(np.int32)
    return SyntheticScene("room", mesh, num_classes, face_labels=labels,
                          class_names=_ROOM_NAMES[:num_classes] if num_classes <= 6 else [])


def make_checker_sphere(radius=1.0, level=2, num_classes=2):
    """Icosphere labelled by an angular checker of period 36 / 2^level degrees in
    (polar angle, azimuth): class borders cut through face interiors."""
    if num_classes < 2:
        raise ConfigError("checker_sphere needs at least 2 classes")
    mesh = make_icosphere(radius, level)
    period = 36.0 / (2 ** level)

    def labels(points):
        p = np.asarray(points, dtype=np.float64)
        r = np.linalg.norm(p, axis=1)
        r = np.where(r == 0.0, 1.0, r)
        polar = np.degrees(np.arccos(np.clip(p[:, 2] / r, -1.0, 1.0)))
        az = np.degrees(np.arctan2(p[:, 1], p[:, 0])) % 360.0
        cell = np.floor(polar / period).astype(np.int64) + np.floor(az / period).astype(np.int64)
        return (cell % num_classes).astype(np.int32)

    return SyntheticScene("checker_sphere", mesh, num_classes, label_fn=labels)


def make_scene(kind, num_classes=None, **params):
    makers = {"cube": (make_cube, 6), "room": (make_room, 6), "checker_sphere": (make_checker_sphere, 2)}
    if kind not in makers:
        raise ConfigError("unknown scene %r (choose from %s)" % (kind, SCENE_KINDS))
    fn, default_c = makers[kind]
    return fn(num_classes=num_classes or default_c, **params)


def render_ground_truth(scene, frame, ids=None):
    """Exact (H, W) int32 labels of one frame, UNKNOWN where no triangle projects."""
    layout = uniform_layout(scene.mesh)
    if ids is None:
        ids = rasterize(scene.mesh, layout, frame)
    out = np.full((ids.height, ids.width), UNKNOWN, dtype=np.int32)
    cov = ids.covered
    if scene.face_labels is not None:
        out[cov] = scene.face_labels[ids.triangle[cov]]
    else:
        out[cov] = scene.label_fn(pixel_world_points(scene.mesh, layout, ids))
    return out


def write_scene_dir(outdir, scene, frames, model, write_gt=True, write_probs=True):
    """mesh.ply, trajectory.txt, palette.txt, gt/<id>.png, probs/<id>.smpb and a
    ready-to-run fuse.cfg under ``outdir``; returns the paths by name."""
    os.makedirs(outdir, exist_ok=True)
    paths = {name: os.path.join(outdir, leaf) for name, leaf in (
        ("mesh", "mesh.ply"), ("trajectory", "trajectory.txt"), ("palette", "palette.txt"), ("gt", "gt"),
        ("probs", "probs"), ("config", "fuse.cfg"))}
    save_ply(paths["mesh"], scene.mesh)
    save_trajectory(paths["trajectory"], frames)
    save_palette(paths["palette"], default_palette(scene.num_classes), scene.class_names or None)
    for flag, key in ((write_gt, "gt"), (write_probs, "probs")):
        if flag:
            os.makedirs(paths[key], exist_ok=True)
    if write_gt or write_probs:
        layout = uniform_layout(scene.mesh)
        for frame in frames:
            gt = render_ground_truth(scene, frame, rasterize(scene.mesh, layout, frame))
            if write_gt:
                write_label_png(os.path.join(paths["gt"], "%d.png" % frame.frame_id), gt, scene.num_classes)
            if write_probs:
                write_probability_image(os.path.join(paths["probs"], "%d.smpb" % frame.frame_id),
                                        corrupt(gt, model, scene.num_classes, frame.frame_id))
    cfg = [("mesh", paths["mesh"]), ("trajectory", paths["trajectory"]), ("predictions", paths["probs"]),
           ("classes", "%d" % scene.num_classes), ("palette", paths["palette"]), ("ground_truth", paths["gt"]),
           ("output", os.path.join(outdir, "fused"))]
    with open(paths["config"], "w", encoding="utf-8") as fh:
        fh.writelines("%s=%s\n" % kv for kv in cfg)
    return paths


__all__ = ["SCENE_KINDS", "NOISE_KINDS", "NoiseModel", "SyntheticScene", "make_cube", "make_room",
           "make_icosphere", "make_checker_sphere", "make_scene", "look_at", "make_orbit_trajectory",
           "render_ground_truth", "corrupt", "write_scene_dir"]

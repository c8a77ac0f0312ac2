"""B200-native label fusion on texel-subdivided triangle meshes (arXiv 2111.11103).

Drop-in for the hot path of the reference package ``texelfuse``: the same
library API (rasterize, compute_pixel_weights, init_texture,
accumulate_frame, finalize, texel_argmax, render_labels, layout helpers),
the same session API (open_session / add_frame / finalize_and_render) and a
batched MeshAnnotation front end, all executing hand-written sm_100a CUDA
kernels through the C ABI in include/texelfuse_b200.h.  There is no CPU
fallback: without the built library and a CUDA device every compute entry
point raises.
"""

from .errors import CapacityError, ConfigError, DataError, TexelFuseError
from .fusion import (
    AGGREGATORS,
    MUL_CLAMP,
    UNKNOWN,
    WEIGHT_MODES,
    ProbabilityTexture,
    accumulate_frame,
    compute_pixel_weights,
    finalize,
    init_texture,
    parse_weight_mode,
    texel_argmax,
    texture_nbytes,
)
from .geometry import (
    MAX_STEPS,
    NEAR_PLANE,
    CameraFrame,
    Intrinsics,
    Mesh,
    TexelLayout,
    build_texel_layout,
    compute_worst_case_areas,
    texel_count,
    texel_id,
    uniform_layout,
)
from .formats import (
    read_probability_header,
    read_probability_image,
    read_texture,
    write_probability_image,
    write_texture,
)
from .meshio import load_mesh, load_trajectory, save_ply, save_trajectory
from .rasterizer import IdImage, dump_debug_images, pixel_world_points, project_point, rasterize
from .renderback import (
    EvalReport,
    colorize_labels,
    default_palette,
    export_colored_mesh,
    load_palette,
    merge_reports,
    pixel_accuracy,
    read_label_png,
    render_labels,
    save_palette,
    select_frames,
    write_label_png,
)
from .synthgen import (
    NoiseModel,
    SyntheticScene,
    corrupt,
    make_orbit_trajectory,
    make_scene,
    render_ground_truth,
    write_scene_dir,
)

__version__ = "0.1.0"


def __getattr__(name):
    # heavier front ends load lazily so `import paper_2111_11103_b200` stays cheap
    if name == "MeshAnnotation":
        from .annotation import MeshAnnotation

        return MeshAnnotation
    if name in ("open_session", "add_frame", "finalize_and_render"):
        from . import session

        return getattr(session, name)
    raise AttributeError(name)


__all__ = [
    "AGGREGATORS", "WEIGHT_MODES", "MUL_CLAMP", "UNKNOWN", "MAX_STEPS", "NEAR_PLANE",
    "CameraFrame", "CapacityError", "ConfigError", "DataError", "IdImage", "Intrinsics", "Mesh",
    "MeshAnnotation", "ProbabilityTexture", "TexelFuseError", "TexelLayout",
    "accumulate_frame", "add_frame", "build_texel_layout", "compute_pixel_weights", "compute_worst_case_areas",
    "finalize", "finalize_and_render", "init_texture", "load_mesh", "load_trajectory", "open_session",
    "parse_weight_mode", "pixel_world_points", "project_point", "rasterize", "render_labels", "save_ply",
    "save_trajectory", "texel_argmax", "texel_count", "texel_id", "texture_nbytes", "uniform_layout",
    "EvalReport", "NoiseModel", "colorize_labels", "corrupt", "default_palette", "export_colored_mesh",
    "load_palette", "make_orbit_trajectory", "merge_reports", "pixel_accuracy", "read_label_png",
    "read_probability_header", "read_probability_image", "read_texture", "save_palette", "select_frames",
    "write_label_png", "write_probability_image", "write_texture", "SyntheticScene", "make_scene",
    "render_ground_truth", "write_scene_dir",
]

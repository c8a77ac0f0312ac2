"""ctypes binding of the C ABI in include/texelfuse_b200.h.

There is no CPU fallback: if the sm_100a library is missing, or no CUDA
device is present, every entry point raises.  Status codes map onto the
reference's exception types (texelfuse/errors.py:4-17).
"""

import ctypes
import os

from .errors import CapacityError, DataError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TFB_LIB") or os.path.join(_PKG, "_lib", "libtexelfuse_b200.so")

TFB_OK, TFB_ERR_DATA, TFB_ERR_CAPACITY, TFB_ERR_STATE, TFB_ERR_CUDA, TFB_ERR_VALUE = range(6)
AGG_IDS = {"sum": 0, "maxsum": 1, "mul": 2}
WMODE_IDS = {"pixels_iid": 0, "images_iid": 1, "blend": 2, "explicit": 3}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t


class TfbScene(ctypes.Structure):
    """Mirror of ``tfb_scene`` (include/texelfuse_b200.h)."""

    _fields_ = [
        ("vertices", _P), ("triangles", _P), ("steps", _P), ("origins", _P), ("offsets", _P),
        ("num_vertices", _I64), ("num_triangles", _I64), ("total_texels", _I64),
        ("clusters", _P), ("num_clusters", _I64),
    ]


_SIGNATURES = {
    "tfb_last_error": ([], ctypes.c_char_p),
    "tfb_version": ([], _I),
    "tfb_set_option": ([_I, _I], _I),
    "tfb_raster_workspace_bytes": ([_I64, _I64, _I, _I, _I, _I64], _SZ),
    "tfb_rasterize": ([_P, _P, _I, _I, _I, _P, _SZ, _I64, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "tfb_rasterize_phases": ([_P, _P, _I, _I, _I, _P, _SZ, _I64, _P, _P, _P, _P, _P, _P, _P, _I, _P], _I),
    "tfb_rows_from_ids": ([_P, _P, _I64, _P, _P, _P, _P], _I),
    "tfb_count_hits": ([_P, _I64, _I, _I64, _P, _P], _I),
    "tfb_clear_hits": ([_P, _I64, _I, _I64, _P, _P], _I),
    "tfb_pixel_weights": ([_P, _I64, _I, _P, _I64, _I, _D, _P, _P], _I),
    "tfb_fuse": ([_P, _I64, _I, _P, _I, _P, _P, _I64, _I, _I, _D, _P, _I, _I64, _P, _P, _P], _I),
    "tfb_fuse_ordered": ([_P, _I64, _I, _P, _I, _P, _P, _I64, _I, _I, _D, _P, _I, _I64, _P, _P, _P, _P, _P], _I),
    "tfb_fuse_order_workspace_bytes": ([_I64, _I, _I64, _I], _SZ),
    "tfb_test_log_f64": ([_P, _P, _I64, _P], _I),
    "tfb_fuse_order": ([_P, _I64, _I, _I64, _I, _P, _SZ, _P, _P, _P], _I),
    "tfb_finalize": ([_P, _I, _I64, _P, _I64, _I, _I, _P, _P, _P, _P], _I),
    "tfb_render": ([_P, _I64, _I, _P, _I64, _P, _P, _P], _I),
    "tfb_probs_argmax": ([_P, _I64, _I, _P, _P], _I),
    "tfb_worst_case_areas": ([_P, _P, _P, _I, _P, _P], _I),
    "tfb_probs_check": ([_P, _I64, _I, _P, _P], _I),
    "tfb_confusion": ([_P, _P, _I64, _I, _P, _P, _P, _P, _P], _I),
    "tfb_face_majority": ([_P, _P, _P, _I64, _I, _P, _P], _I),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path=LIB_PATH):
    """Load the shared library (no CUDA device needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            "texelfuse_b200 CUDA extension not built (%s missing); run "
            "`python -m paper_2111_11103_b200.build`" % path)
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error():
    return load().tfb_last_error().decode("utf-8", "replace")


def check(rc, what=""):
    if rc == TFB_OK:
        return
    msg = last_error() or what
    if rc == TFB_ERR_DATA:
        raise DataError(msg)
    if rc == TFB_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == TFB_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc


def ptr(t):
    """Device (or host) address of a torch tensor / None → NULL."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def ptr_array(addrs):
    """Host array of device pointers (tfb_fuse's per-frame probability maps)."""
    arr = (ctypes.c_void_p * max(len(addrs), 1))(*[int(a) for a in addrs])
    return ctypes.cast(arr, ctypes.c_void_p), arr


def stream_handle(stream=None):
    """cudaStream_t of ``stream``, else of the current stream of the current device
    (callers that own tensors on another device enter ``torch.cuda.device`` first)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


PINNED_READBACK_LIMIT = 64 << 20


def host_copy(t):
    """NumPy copy of a device tensor, read back through page-locked memory from torch's
    caching host allocator (a DMA at full PCIe rate, no allocation after warm-up, instead
    of the driver's pageable staging); the array keeps its pinned buffer alive.  Large
    tensors (> 64 MB: per-call pinned allocations would be costly and hog host memory) and
    host tensors take the plain copy."""
    import torch

    if not t.is_cuda or t.numel() * t.element_size() > PINNED_READBACK_LIMIT:
        return t.detach().cpu().numpy()
    with torch.cuda.device(t.device):
        pinned = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        pinned.copy_(t.detach(), non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
    return pinned.numpy()


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("texelfuse_b200 needs a CUDA device (B200, sm_100a); none is available")
    load()

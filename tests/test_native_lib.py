"""The C-ABI library loads and exports every symbol include/texelfuse_b200.h
declares; argument validation and error mapping work without a GPU; the
product path refuses to run without a CUDA device (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2111_11103_b200 import _native as N
from paper_2111_11103_b200.errors import DataError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "texelfuse_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return set(re.findall(r"\b(tfb_\w+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_symbols() == set(N.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.tfb_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_query_is_host_only():
    lib = N.load()
    a = lib.tfb_raster_workspace_bytes(151686, 299568, 640, 480, 1, 0)
    b = lib.tfb_raster_workspace_bytes(151686, 299568, 640, 480, 8, 0)
    assert a > 299568 * 2 * 96 and b > 7 * a  # 96-byte records at 2 slots per triangle


def test_argument_errors_map_to_reference_exceptions():
    lib = N.load()
    rc = lib.tfb_fuse(ctypes.c_void_p(16), 4, 1, ctypes.c_void_p(16), 3, None, None, 10, 7, 0, 0.0,
                      ctypes.c_void_p(16), 0, 4, ctypes.c_void_p(16), None, None)
    assert rc == N.TFB_ERR_VALUE
    assert "aggregator" in N.last_error()
    with pytest.raises(ValueError):
        N.check(rc)
    rc = lib.tfb_rasterize(None, None, 1, 64, 64, None, 0, 0, None, None, None, None, None, None, None, None)
    assert rc == N.TFB_ERR_DATA
    with pytest.raises(DataError):
        N.check(rc)
    rc = lib.tfb_fuse(ctypes.c_void_p(16), 4, 1, ctypes.c_void_p(16), 3, None, None, 10, 0, 1, 0.0,
                      ctypes.c_void_p(16), 0, 4, ctypes.c_void_p(16), None, None)
    assert rc == N.TFB_ERR_DATA and "hit counts" in N.last_error()
    # optional output planes come in groups (checked before any device work)
    scene = N.TfbScene(None, None, None, None, None, 3, 1, 1, None, 0)
    dev = ctypes.c_void_p(256)
    rc = lib.tfb_rasterize(ctypes.byref(scene), dev, 1, 64, 64, dev, 1 << 30, 0, dev, None, dev, None, None, None,
                           None, None)
    assert rc == N.TFB_ERR_VALUE and "together" in N.last_error()
    rc = lib.tfb_rasterize(ctypes.byref(scene), dev, 1, 64, 64, dev, 1 << 30, 0, dev, None, None, None, dev, dev,
                           None, None)
    assert rc == N.TFB_ERR_VALUE and "together" in N.last_error()


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2111_11103_b200 import Mesh, rasterize, uniform_layout
    from paper_2111_11103_b200.geometry import CameraFrame, Intrinsics

    mesh = Mesh.from_arrays(np.array([[0, 0, 1], [1, 0, 1], [0, 1, 1.0]]), np.array([[0, 1, 2]]))
    fr = CameraFrame(0, Intrinsics(8, 8, 4, 4, 8, 8), np.eye(3), np.zeros(3))
    with pytest.raises(RuntimeError, match="CUDA"):
        rasterize(mesh, uniform_layout(mesh), fr)

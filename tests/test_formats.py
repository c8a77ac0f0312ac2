"""SMPB / SMTX readers and writers against files written by the reference's
own writers (tests/golden/make_golden_formats.py), byte for byte, plus the
reference tests' error cases (test_formats.py).  SMPB pixel validation runs
on the GPU (tfb_probs_check), so those tests are marked gpu."""

import os
import struct

import numpy as np
import pytest

from paper_2111_11103_b200 import DataError, TexelLayout
from paper_2111_11103_b200 import formats as F

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")


def _golden_layout():
    d = np.load(os.path.join(G, "texture.npz"))
    layout = TexelLayout(steps=d["steps"], origins=d["origins"], offsets=d["offsets"],
                         total_texels=int(len(d["rows"])))
    return layout, d


def test_smpb_writer_bytes_match_reference(tmp_path):
    for name in ("probs_12x17x5", "probs_3x4x40"):
        p = np.load(os.path.join(G, name + ".npy"))
        out = tmp_path / (name + ".smpb")
        F.write_probability_image(out, p)
        assert out.read_bytes() == open(os.path.join(G, name + ".smpb"), "rb").read()
        assert F.read_probability_header(out) == p.shape


def test_smpb_header_errors(tmp_path):
    path = tmp_path / "x.smpb"
    with pytest.raises(DataError):
        F.write_probability_image(path, np.zeros((4, 4), dtype=np.float32))
    path.write_bytes(b"JUNK" + b"\x00" * 32)
    with pytest.raises(DataError, match="magic"):
        F.read_probability_header(path)
    data = open(os.path.join(G, "probs_12x17x5.smpb"), "rb").read()
    path.write_bytes(data[:4] + struct.pack("<I", 9) + data[8:])
    with pytest.raises(DataError, match="version"):
        F.read_probability_header(path)
    path.write_bytes(data[:4] + struct.pack("<IIII", 1, 0, 4, 4))
    with pytest.raises(DataError, match="invalid dimensions"):
        F.read_probability_header(path)
    with pytest.raises(DataError, match="cannot read prediction"):
        F.read_probability_header(tmp_path / "missing.smpb")


def test_smtx_writer_bytes_match_reference(tmp_path):
    layout, d = _golden_layout()
    out = tmp_path / "t.smtx"
    F.write_texture(out, layout, d["rows"], d["counts"], unobserved=d["unobserved"])
    assert out.read_bytes() == open(os.path.join(G, "texture.smtx"), "rb").read()


def test_smtx_reader_matches_reference_file():
    layout, d = _golden_layout()
    back, rows, counts = F.read_texture(os.path.join(G, "texture.smtx"))
    np.testing.assert_array_equal(back.steps, layout.steps)
    np.testing.assert_array_equal(back.origins, layout.origins)
    np.testing.assert_array_equal(back.offsets, layout.offsets)
    assert back.total_texels == layout.total_texels
    np.testing.assert_array_equal(rows, d["rows"])
    expect = d["counts"].copy()
    expect[d["unobserved"]] = 0
    np.testing.assert_array_equal(counts, expect)
    assert counts.dtype == np.int64 and rows.dtype == np.float32


def test_smtx_errors(tmp_path):
    layout = TexelLayout(steps=np.array([1]), origins=np.array([0]), offsets=np.array([0]), total_texels=1)
    rows = np.array([[0.5, 0.5]], dtype=np.float32)
    path = tmp_path / "t.smtx"
    F.write_texture(path, layout, rows, np.array([1]))
    raw = path.read_bytes()
    assert struct.unpack_from("<I", raw, 0)[0] == 1 and raw[9:13] == b"SMTX"
    broken = bytearray(raw)
    broken[9:13] = b"NOPE"
    path.write_bytes(bytes(broken))
    with pytest.raises(DataError, match="magic"):
        F.read_texture(path)
    path.write_bytes(raw[:10])
    with pytest.raises(DataError):
        F.read_texture(path)
    path.write_bytes(struct.pack("<I", 10 ** 6) + raw[4:])
    with pytest.raises(DataError, match="implausible"):
        F.read_texture(path)
    bad = bytearray(raw)
    bad[4:8] = struct.pack("<I", 0)
    path.write_bytes(bytes(bad))
    with pytest.raises(DataError, match="non-positive steps"):
        F.read_texture(path)
    bad = bytearray(raw)
    bad[8] = 3
    path.write_bytes(bytes(bad))
    with pytest.raises(DataError, match="origin vertex"):
        F.read_texture(path)
    bad = bytearray(raw)
    bad[17:25] = struct.pack("<Q", 2)
    path.write_bytes(bytes(bad))
    with pytest.raises(DataError, match="implies"):
        F.read_texture(path)
    path.write_bytes(raw[:-2])
    with pytest.raises(DataError, match="truncated observation counts"):
        F.read_texture(path)
    path.write_bytes(raw[:-6])
    with pytest.raises(DataError, match="truncated texture rows"):
        F.read_texture(path)
    with pytest.raises(DataError, match="do not match"):
        F.write_texture(path, layout, np.zeros((2, 2), np.float32), np.zeros(2))
    with pytest.raises(DataError, match="counts shape"):
        F.write_texture(path, layout, rows, np.zeros(3))
    with pytest.raises(DataError, match="cannot read texture"):
        F.read_texture(tmp_path / "missing.smtx")


@pytest.mark.gpu
def test_smpb_read_validates_on_device(tmp_path):
    import torch

    for name in ("probs_12x17x5", "probs_3x4x40"):
        p = np.load(os.path.join(G, name + ".npy"))
        back = F.read_probability_image(os.path.join(G, name + ".smpb"))
        assert back.dtype == np.float32
        np.testing.assert_array_equal(back, p)
        dev = F.read_probability_image(os.path.join(G, name + ".smpb"), device="cuda")
        assert dev.is_cuda and dev.dtype == torch.float32
        np.testing.assert_array_equal(dev.cpu().numpy(), p)
        out = torch.empty(p.shape, dtype=torch.float32, device="cuda")
        F.read_probability_image(os.path.join(G, name + ".smpb"), out=out)
        np.testing.assert_array_equal(out.cpu().numpy(), p)


@pytest.mark.gpu
def test_smpb_device_validation_errors(tmp_path):
    path = tmp_path / "x.smpb"
    F.write_probability_image(path, np.full((2, 2, 3), 0.5, dtype=np.float32))
    with pytest.raises(DataError, match="sum to 1 \\(max error 0.5\\)"):
        F.read_probability_image(path)
    F.write_probability_image(path, np.array([[[1.2, -0.2, 0.0]]], dtype=np.float32))
    with pytest.raises(DataError, match="negative"):
        F.read_probability_image(path)
    # a NaN passes like in the reference (np.min / the sums propagate NaN, NaN > tol is False)
    nanp = np.full((1, 1, 2), 0.5, dtype=np.float32)
    nanp[0, 0, 0] = np.nan
    F.write_probability_image(path, nanp)
    assert np.isnan(F.read_probability_image(path)[0, 0, 0])
    # sums are float64: 1 - 1e-4 < s < 1 + 1e-4 passes, 1 + 2e-4 does not
    rng = np.random.default_rng(3)
    p = rng.random((64, 64, 40)).astype(np.float32)
    p /= p.sum(axis=2, keepdims=True)
    F.write_probability_image(path, p)
    F.read_probability_image(path, device="cuda")
    p[5, 7, 3] += np.float32(2e-4)
    F.write_probability_image(path, p)
    with pytest.raises(DataError, match="max error 0.0002"):
        F.read_probability_image(path, device="cuda")
    data = path.read_bytes()
    path.write_bytes(data[:-8])
    with pytest.raises(DataError, match="truncated"):
        F.read_probability_image(path)


@pytest.mark.gpu
def test_texture_written_from_device(tmp_path):
    import torch

    layout, d = _golden_layout()
    rows = torch.as_tensor(d["rows"]).cuda()
    counts = torch.as_tensor(d["counts"]).to(torch.int32).cuda()
    unobs = torch.as_tensor(d["unobserved"]).cuda()
    out = tmp_path / "t.smtx"
    F.write_texture(out, layout, rows, counts, unobserved=unobs)
    assert out.read_bytes() == open(os.path.join(G, "texture.smtx"), "rb").read()

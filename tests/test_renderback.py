"""renderback helpers (reference renderback.py): frame selection, EvalReport,
reports, label PNGs, palettes, colorizing (CPU); pixel_accuracy and the
colored-mesh face vote run on the GPU (tfb_confusion, tfb_face_majority)."""

import json

import numpy as np
import pytest

from paper_2111_11103_b200 import DataError, Mesh, TexelLayout
from paper_2111_11103_b200.renderback import (
    UNKNOWN, EvalReport, colorize_labels, default_palette, export_colored_mesh, load_palette, merge_reports,
    pixel_accuracy, read_label_png, save_palette, select_frames, write_label_png, write_report)


def test_select_frames():
    assert select_frames(10, 1.0) == list(range(10))
    assert select_frames(10, 0.5) == [0, 2, 4, 6, 8]
    assert select_frames(7, 0.01) == [0]
    assert select_frames(3, 0.9) == [0, 1, 2]
    prev = 0
    for frac in (0.1, 0.3, 0.6, 1.0):
        n = len(select_frames(50, frac))
        assert n >= prev
        prev = n
    with pytest.raises(ValueError):
        select_frames(10, 0.0)
    with pytest.raises(ValueError):
        select_frames(0, 0.5)


def test_eval_report_merge_lines_json(tmp_path):
    a = EvalReport(2, np.array([[3, 1], [0, 2]]), np.array([1, 0]), ignored=4)
    b = EvalReport(2, np.array([[1, 0], [1, 1]]), np.array([0, 2]), ignored=1)
    m = merge_reports([a, b])
    assert m.evaluated == 12 and m.correct == 7 and m.ignored == 5
    assert m.accuracy == pytest.approx(7 / 12)
    lines = m.to_lines("fused_")
    assert lines[0] == "fused_evaluated 12" and lines[-1] == "fused_accuracy 0.583333"
    d = m.to_json_dict()
    assert d["confusion"] == [[4, 1], [1, 3]] and d["unknown_by_class"] == [1, 2]
    txt, js = tmp_path / "r.txt", tmp_path / "r.json"
    write_report(txt, js, [("", {"frames_used": 3}), ("fused_", m)])
    assert "frames_used 3" in txt.read_text() and "fused_correct 7" in txt.read_text()
    data = json.loads(js.read_text())
    assert data["frames_used"] == 3 and data["fused"]["evaluated"] == 12
    with pytest.raises(DataError):
        a.merge(EvalReport(3))
    with pytest.raises(DataError):
        EvalReport(2, np.zeros((3, 3)))
    assert EvalReport(4).accuracy == 0.0


def test_label_png_round_trips_and_errors(tmp_path):
    small = np.array([[0, 1, 7], [UNKNOWN, 254, 300]], dtype=np.int32)  # 300 >= c: stored as sentinel
    write_label_png(tmp_path / "a.png", small, num_classes=255)
    back = read_label_png(tmp_path / "a.png")
    expect = small.copy()
    expect[1, 2] = UNKNOWN
    np.testing.assert_array_equal(back, expect)
    big = np.array([[0, 300, 64999], [UNKNOWN, 5, 1000]], dtype=np.int64)
    write_label_png(tmp_path / "b.png", big, num_classes=65000)
    np.testing.assert_array_equal(read_label_png(tmp_path / "b.png"), big)
    with pytest.raises(DataError):
        write_label_png(tmp_path / "c.png", np.zeros((2, 2)), num_classes=70000)
    with pytest.raises(DataError):
        write_label_png(tmp_path / "c.png", np.zeros(4), num_classes=3)
    from PIL import Image

    Image.new("RGB", (3, 3)).save(tmp_path / "rgb.png")
    with pytest.raises(DataError):
        read_label_png(tmp_path / "rgb.png")
    with pytest.raises(DataError):
        read_label_png(tmp_path / "missing.png")


def test_palettes_and_colorize(tmp_path):
    colors = default_palette(7)
    assert colors.shape == (7, 3) and len({tuple(c) for c in colors}) == 7
    save_palette(tmp_path / "p.txt", colors, names=list("abcdefg"))
    back, names = load_palette(tmp_path / "p.txt")
    np.testing.assert_array_equal(back, colors)
    assert names == list("abcdefg")
    (tmp_path / "q.txt").write_text("# sparse\n2 10 20 30 wall\n")
    back, names = load_palette(tmp_path / "q.txt")
    assert back.shape == (3, 3) and names == ["class_0", "class_1", "wall"]
    for bad, what in (("1 1 1 1 a\n1 2 2 2 b\n", "duplicate"), ("0 256 0 0\n", "range"), ("zzz\n", "expected"),
                      ("-1 0 0 0\n", "negative"), ("", "empty")):
        (tmp_path / "bad.txt").write_text(bad)
        with pytest.raises(DataError, match=what):
            load_palette(tmp_path / "bad.txt")
    img = colorize_labels(np.array([[0, UNKNOWN, 6, 9]]), colors)
    np.testing.assert_array_equal(img[0, 0], colors[0])
    np.testing.assert_array_equal(img[0, 1], [128, 128, 128])
    np.testing.assert_array_equal(img[0, 2], colors[6])
    np.testing.assert_array_equal(img[0, 3], [128, 128, 128])


@pytest.mark.gpu
def test_pixel_accuracy_semantics():
    rep = pixel_accuracy(np.array([[0, 1, 1, 0]]), np.array([[0, 1, 0, 0]]), 2)
    assert rep.evaluated == 4 and rep.correct == 3 and rep.ignored == 0
    assert rep.confusion.tolist() == [[2, 1], [0, 1]]
    # reference pixels UNKNOWN / out of range / ignored are skipped; predictions
    # outside [0, c) count as unknown (evaluated, wrong)
    pred = np.array([[0, UNKNOWN, 5, 2, 1, 2]])
    ref = np.array([[0, 0, 1, UNKNOWN, 7, 2]])
    rep = pixel_accuracy(pred, ref, 3, ignore=[2])
    assert rep.ignored == 3 and rep.evaluated == 3 and rep.correct == 1
    assert rep.unknown_pred.tolist() == [1, 1, 0]
    with pytest.raises(DataError):
        pixel_accuracy(np.zeros((2, 2)), np.zeros((2, 3)), 2)
    # a noisy prediction scores its noise rate
    rng = np.random.default_rng(0)
    ref = rng.integers(0, 5, size=(64, 80))
    pred = ref.copy()
    flip = rng.random(ref.shape) < 0.3
    pred[flip] = (pred[flip] + 1) % 5
    assert pixel_accuracy(pred, ref, 5).accuracy == pytest.approx(1 - flip.mean())
    # more classes than the shared-memory histogram holds (global-atomic path)
    c = 100
    ref = rng.integers(0, c, size=(50, 50))
    pred = np.where(rng.random(ref.shape) < 0.5, ref, rng.integers(0, c, size=ref.shape))
    rep = pixel_accuracy(pred, ref, c)
    np.testing.assert_array_equal(rep.confusion, np.bincount(ref.ravel() * c + pred.ravel(),
                                                             minlength=c * c).reshape(c, c))


@pytest.mark.gpu
def test_export_colored_mesh_vote(tmp_path):
    verts = np.array([[0, 0, 1], [1, 0, 1], [0, 1, 1], [1, 1, 1], [2, 0, 1]], dtype=np.float64)
    tris = np.array([[0, 1, 2], [1, 3, 2], [1, 4, 3]], dtype=np.int32)
    mesh = Mesh.from_arrays(verts, tris)
    steps = np.array([1, 4, 2], dtype=np.int32)  # 1, 10, 3 texels
    offsets = np.array([0, 1, 11], dtype=np.int64)
    layout = TexelLayout(steps=steps, origins=np.zeros(3, np.int8), offsets=offsets, total_texels=14)
    colors = default_palette(5)
    labels = np.full(14, UNKNOWN, dtype=np.int64)
    labels[0] = 3                   # face 0: one texel of class 3
    labels[1:4] = 4                 # face 1: 3 x class 4, 3 x class 1 (tie -> lower class), rest unknown
    labels[4:7] = 1
    labels[11] = 9                  # face 2: only an out-of-range label -> unobserved gray
    path = tmp_path / "m.ply"
    export_colored_mesh(path, mesh, layout, labels, colors)
    raw = path.read_bytes()
    end = raw.index(b"end_header\n") + len(b"end_header\n")
    nv = int([ln for ln in raw[:end].decode().splitlines() if ln.startswith("element vertex")][0].split()[-1])
    rec = np.dtype([("n", "u1"), ("idx", "<i4", (3,)), ("rgb", "u1", (3,))])
    rgb = np.frombuffer(raw[end + nv * 12:], dtype=rec, count=3)["rgb"]
    np.testing.assert_array_equal(rgb[0], colors[3])
    np.testing.assert_array_equal(rgb[1], colors[1])
    np.testing.assert_array_equal(rgb[2], [128, 128, 128])
    with pytest.raises(DataError):
        export_colored_mesh(path, mesh, layout, labels[:5], colors)

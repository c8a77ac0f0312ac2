"""The GPU-backed CLI (paper_2111_11103_b200/cli.py) against a run of the
reference CLI on the same synthetic scene (tests/golden/cli, see its README):
texture.smtx, label PNGs, reports, the colored mesh, render and eval outputs.
Configuration handling and the fail-fast data checks run without a GPU."""

import os
import shutil

import numpy as np
import pytest

from paper_2111_11103_b200 import cli, formats
from paper_2111_11103_b200.errors import ConfigError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
SCENE = os.path.join(G, "scene")
REF = os.path.join(G, "ref")


def _fuse_args(out, **extra):
    args = ["mesh=" + os.path.join(SCENE, "mesh.ply"), "trajectory=" + os.path.join(SCENE, "trajectory.txt"),
            "predictions=" + os.path.join(SCENE, "probs"), "classes=5",
            "palette=" + os.path.join(SCENE, "palette.txt"), "ground_truth=" + os.path.join(SCENE, "gt"),
            "output=" + str(out)]
    return args + ["%s=%s" % kv for kv in extra.items()]


def test_config_parsing(tmp_path):
    assert cli.parse_pairs(["a=1", "--b", "2", "--c-d=3", "help"]) == {"a": "1", "b": "2", "c_d": "3",
                                                                      "help": "true"}
    cfg = tmp_path / "x.cfg"
    cfg.write_text("# comment\ngamma = 0.4\nclasses=3\n")
    assert cli.resolve(["config=%s" % cfg, "classes=7"]) == {"gamma": "0.4", "classes": "7"}
    with pytest.raises(ConfigError):
        cli.parse_pairs(["novalue"])
    with pytest.raises(ConfigError):
        cli.parse_pairs(["--dangling"])
    cfg.write_text("broken line\n")
    with pytest.raises(ConfigError, match="expected key=value"):
        cli.resolve(["config=%s" % cfg])


def test_exit_codes_without_gpu(tmp_path, capsys):
    assert cli.main([]) == 2
    assert cli.main(["--help"]) == 0
    assert cli.main(["bogus"]) == 2
    assert cli.main(["synth"]) == 2
    assert cli.main(["fuse", "mesh=x"]) == 2  # missing keys
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", bogus_key=1)) == 2
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", classes=1)) == 2
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", aggregator="nope")) == 2
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", fallback="x")) == 2
    # wrong class count in the predictions: caught by the header check, before any GPU work
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", classes=6)) == 3
    assert "has 5 classes, config says 6" in capsys.readouterr().err
    empty = tmp_path / "probs"
    empty.mkdir()
    args = _fuse_args(tmp_path / "o")
    args[2] = "predictions=%s" % empty
    assert cli.main(["fuse"] + args) == 3
    assert cli.main(["eval", "labels=x", "ground_truth=%s" % (tmp_path / "none"), "classes=5"]) == 3


@pytest.mark.gpu
def test_fuse_matches_reference_cli(tmp_path):
    out = tmp_path / "fused"
    assert cli.main(["fuse"] + _fuse_args(out, export_mesh="true")) == 0
    ref = os.path.join(REF, "fuse")
    # texture: identical layout table and counts, rows within float64-accumulation rounding
    lr, rr, cr = formats.read_texture(os.path.join(ref, "texture.smtx"))
    lo, ro, co = formats.read_texture(out / "texture.smtx")
    np.testing.assert_array_equal(lo.steps, lr.steps)
    np.testing.assert_array_equal(lo.origins, lr.origins)
    np.testing.assert_array_equal(co, cr)
    np.testing.assert_allclose(ro, rr, rtol=0, atol=1e-6)
    raw_o, raw_r = (open(p, "rb").read() for p in (out / "texture.smtx", os.path.join(ref, "texture.smtx")))
    assert raw_o[:4 + 5 * lr.num_triangles + 20] == raw_r[:4 + 5 * lr.num_triangles + 20]
    # reports and labels
    assert (out / "report.txt").read_text() == open(os.path.join(ref, "report.txt")).read()
    from paper_2111_11103_b200.renderback import read_label_png

    for name in sorted(os.listdir(os.path.join(ref, "labels"))):
        np.testing.assert_array_equal(read_label_png(out / "labels" / name),
                                      read_label_png(os.path.join(ref, "labels", name)))
    assert (out / "labeled_mesh.ply").read_bytes() == open(os.path.join(ref, "labeled_mesh.ply"), "rb").read()
    conf = dict(line.split("=", 1) for line in (out / "config.txt").read_text().splitlines())
    conf_ref = dict(line.split("=", 1) for line in open(os.path.join(ref, "config.txt")).read().splitlines())
    paths = {"output", "mesh", "trajectory", "predictions", "palette", "ground_truth"}
    assert set(conf) == set(conf_ref)
    for k in set(conf_ref) - paths:
        assert conf[k] == conf_ref[k], k


@pytest.mark.gpu
def test_fuse_float32_accumulator_and_unknown_fallback(tmp_path):
    out = tmp_path / "f32"
    assert cli.main(["fuse"] + _fuse_args(out, accum="float32", fallback="unknown", batch=4)) == 0
    lr, rr, cr = formats.read_texture(os.path.join(REF, "fuse", "texture.smtx"))
    _, ro, co = formats.read_texture(out / "texture.smtx")
    np.testing.assert_array_equal(co, cr)
    np.testing.assert_allclose(ro, rr, rtol=0, atol=2e-5)


@pytest.mark.gpu
def test_render_and_eval_match_reference_cli(tmp_path):
    out = tmp_path / "render"
    assert cli.main(["render", "texture=" + os.path.join(REF, "fuse", "texture.smtx"),
                     "mesh=" + os.path.join(SCENE, "mesh.ply"), "trajectory=" + os.path.join(SCENE, "trajectory.txt"),
                     "output=%s" % out, "color=true", "palette=" + os.path.join(SCENE, "palette.txt")]) == 0
    ref = os.path.join(REF, "render")
    for name in sorted(os.listdir(ref)):
        from PIL import Image

        a = np.asarray(Image.open(out / name))
        b = np.asarray(Image.open(os.path.join(ref, name)))
        np.testing.assert_array_equal(a, b, err_msg=name)
    labels = tmp_path / "labels"
    shutil.copytree(os.path.join(REF, "fuse", "labels"), labels)
    ev = tmp_path / "eval"
    assert cli.main(["eval", "labels=%s" % labels, "ground_truth=" + os.path.join(SCENE, "gt"), "classes=5",
                     "output=%s" % ev, "ignore=0"]) == 0
    assert (ev / "report.txt").read_text() == open(os.path.join(REF, "eval", "report.txt")).read()
    assert (ev / "report.json").read_text() == open(os.path.join(REF, "eval", "report.json")).read()


def test_deterministic_needs_fixed_accumulator(tmp_path):
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", deterministic="true", accum="float32")) == 2
    assert cli.main(["fuse"] + _fuse_args(tmp_path / "o", accum="float16")) == 2


@pytest.mark.gpu
def test_criterion_09_deterministic_reruns_are_byte_identical(tmp_path):
    """test_acceptance.py:373-399: two `fuse ... deterministic=true` runs write
    byte-identical texture.smtx and label PNGs (fixed64 accumulator)."""
    outs = []
    for name in ("a", "b"):
        out = tmp_path / name
        assert cli.main(["fuse"] + _fuse_args(out, aggregator="mul", deterministic="true", batch=3 if name == "a"
                                              else 64)) == 0
        outs.append(out)
    a, b = outs
    assert (a / "texture.smtx").read_bytes() == (b / "texture.smtx").read_bytes()
    pngs = sorted(os.listdir(a / "labels"))
    assert pngs
    for f in pngs:
        assert (a / "labels" / f).read_bytes() == (b / "labels" / f).read_bytes()

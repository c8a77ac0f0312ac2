"""Checkpoint / resume of a fusion job (MeshAnnotation.save_checkpoint /
load_checkpoint; SURVEY §3 "checkpoint / resume": the accumulator is a sum
monoid, so resuming means adding the remaining frames)."""

import numpy as np
import pytest
import torch

from paper_2111_11103_b200 import DataError, Mesh, MeshAnnotation, uniform_layout
from paper_2111_11103_b200.geometry import Intrinsics
from paper_2111_11103_b200.synth import make_room, random_room_trajectory, softmax_maps

pytestmark = pytest.mark.gpu


def _job(mesh, layout, frames, probs, agg, accum_dtype):
    return MeshAnnotation(mesh, layout, num_classes=probs[0].shape[-1], aggregator=agg, accum_dtype=accum_dtype,
                          max_batch=4)


@pytest.mark.parametrize("agg,accum_dtype", [("mul", "float32"), ("sum", "float64")])
def test_checkpoint_resume_equals_one_job(tmp_path, agg, accum_dtype):
    v, t = make_room((6.0, 5.0, 3.0), 12)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    intr = Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96)
    frames = random_room_trajectory(10, intr, seed=4)
    probs = list(softmax_maps(10, 96, 128, 7, seed=2))
    whole = _job(mesh, layout, frames, probs, agg, accum_dtype)
    whole.add_batch(probs, frames)
    c = probs[0].shape[-1]
    ref_acc = whole.texture._accum[:, :c].double().cpu().numpy()
    ref_cnt = whole.texture._counts.cpu().numpy()

    first = _job(mesh, layout, frames, probs, agg, accum_dtype)
    first.add_batch(probs[:6], frames[:6])
    path = tmp_path / "ckpt.npz"
    first.save_checkpoint(path)
    resumed = _job(mesh, layout, frames, probs, agg, accum_dtype)
    resumed.load_checkpoint(path)
    assert resumed.frames_added == 6
    resumed.add_batch(probs[6:], frames[6:])
    acc = resumed.texture._accum[:, :c].double().cpu().numpy()
    tol = 1e-5 if accum_dtype == "float32" else 1e-12
    np.testing.assert_allclose(acc, ref_acc, rtol=tol, atol=tol * np.abs(ref_acc).max())
    np.testing.assert_array_equal(resumed.texture._counts.cpu().numpy(), ref_cnt)
    np.testing.assert_allclose(resumed.get(host=True), whole.get(host=True), rtol=1e-4, atol=1e-6)


def test_checkpoint_mismatch_raises(tmp_path):
    v, t = make_room((6.0, 5.0, 3.0), 6)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    a = MeshAnnotation(mesh, layout, num_classes=5, aggregator="sum")
    path = tmp_path / "a.npz"
    a.save_checkpoint(path)
    with pytest.raises(DataError):
        MeshAnnotation(mesh, layout, num_classes=6, aggregator="sum").load_checkpoint(path)
    with pytest.raises(DataError):
        MeshAnnotation(mesh, layout, num_classes=5, aggregator="mul").load_checkpoint(path)
    with pytest.raises(DataError):
        MeshAnnotation(mesh, uniform_layout(mesh, 2), num_classes=5, aggregator="sum").load_checkpoint(path)
    a.labels()
    with pytest.raises(RuntimeError):
        a.save_checkpoint(path)

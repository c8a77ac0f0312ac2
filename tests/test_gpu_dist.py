"""MeshAnnotation.finalize_distributed on one GPU (world size 1: the slice
finalize is the whole texture) equals labels() — the per-slice tfb_finalize
call that dist.reduce_scatter_finalize makes on every rank.  The multi-rank
exchange itself is covered by tests/test_dist_gloo.py."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("agg", ["sum", "mul"])
def test_finalize_distributed_single_rank(agg):
    import torch

    from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout
    from paper_2111_11103_b200.geometry import Intrinsics
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, softmax_maps

    v, t = make_room((6.0, 5.0, 3.0), 24)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 2)
    frames = random_room_trajectory(6, Intrinsics(100.0, 100.0, 63.5, 47.5, 128, 96), seed=4)
    probs = softmax_maps(6, 96, 128, 12, seed=1)
    a = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, max_batch=6)
    b = MeshAnnotation(mesh, layout, num_classes=12, aggregator=agg, max_batch=6)
    a.add_batch(probs, frames)
    b.add_batch(probs, frames)
    got = a.finalize_distributed()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), b.labels(host=True))
    np.testing.assert_array_equal(a.render(frames, host=True), b.render(frames, host=True))
    with pytest.raises(RuntimeError):
        a.finalize_distributed()

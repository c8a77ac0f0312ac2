"""Multi-rank host logic on CPU (gloo, world_size 2): frame sharding plus ONE sum
all-reduce of (accumulator, counts) reproduces the single-rank texture.  The
per-rank fold here is the CPU oracle (the GPU fold is covered by the parity
tests); what is under test is paper_2111_11103_b200.dist."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene():
    z = np.load(os.path.join(GOLD, "cfg1.npz"))
    from paper_2111_11103_b200.synth import NoiseModel, corrupt

    c = int(z["num_classes"])
    model = NoiseModel("flip", epsilon=0.3, q=0.8, seed=1)
    probs = [corrupt(z["gt"][f].astype(np.int32), model, c, f) for f in range(len(z["cams"]))]
    return z, probs


def _fold(z, probs, frames, agg):
    import oracle as O

    n_x, c = int(z["total_texels"]), int(z["num_classes"])
    acc = np.zeros((n_x, c))
    cnt = np.zeros(n_x, np.int64)
    for f in frames:
        w = O.compute_pixel_weights(z["tri"][f], z["texel"][f], "images_iid")
        O.accumulate_frame(acc, cnt, z["offsets"], z["tri"][f], z["texel"][f], probs[f], w, agg)
    return acc, cnt


def _worker(rank, world, port, agg, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2111_11103_b200 import dist as D

    r, w, _ = D.init_from_env("gloo")
    assert (r, w) == (rank, world)
    z, probs = _scene()
    mine = D.shard_frames(list(range(len(z["cams"]))))
    acc, cnt = _fold(z, probs, mine, agg)
    ta, tc = torch.from_numpy(acc), torch.from_numpy(cnt)
    D.allreduce_sum_([ta, tc])
    if rank == 0:
        np.save(out + "_acc.npy", ta.numpy())
        np.save(out + "_cnt.npy", tc.numpy())
        np.save(out + "_mine.npy", np.array(mine))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("agg", ["sum", "mul"])
def test_two_rank_shards_plus_allreduce_equal_single_rank(tmp_path, agg):
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, _free_port(), agg, out), nprocs=2, join=True)
    z, probs = _scene()
    acc1, cnt1 = _fold(z, probs, range(len(z["cams"])), agg)
    np.testing.assert_array_equal(np.load(out + "_cnt.npy"), cnt1)
    np.testing.assert_allclose(np.load(out + "_acc.npy"), acc1, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(np.load(out + "_mine.npy"), np.arange(10))
    import oracle as O

    rows, unobs = O.finalize(np.load(out + "_acc.npy"), cnt1, agg)
    ref_rows, ref_unobs = O.finalize(acc1, cnt1, agg)
    np.testing.assert_array_equal(O.texel_argmax(rows, unobs), O.texel_argmax(ref_rows, ref_unobs))


def test_shard_bounds_partition():
    from paper_2111_11103_b200.dist import shard_bounds

    for n in (0, 1, 7, 2000):
        for p in (1, 2, 3, 8):
            got = [shard_bounds(n, r, p) for r in range(p)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(p - 1))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _rs_worker(rank, world, port, agg, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import oracle as O
    from paper_2111_11103_b200 import dist as D

    D.init_from_env("gloo")
    z, probs = _scene()
    mine = D.shard_frames(list(range(len(z["cams"]))))
    acc, cnt = _fold(z, probs, mine, agg)

    def finalize_slice(a, c):  # stands in for tfb_finalize on the rank's GPU
        rows, unobs = O.finalize(a.numpy(), c.numpy(), agg)
        return torch.from_numpy(O.texel_argmax(rows, unobs).astype(np.int32))

    ta, tc = torch.from_numpy(acc), torch.from_numpy(cnt.astype(np.int32))  # the product's count dtype
    (sa, sc), (lo, hi) = D.reduce_scatter_rows([ta, tc])
    np.save(out + "_slice%d.npy" % rank, np.concatenate([sa.numpy(), sc.numpy()[:, None]], axis=1))
    np.save(out + "_bounds%d.npy" % rank, np.array([lo, hi]))
    labels = D.reduce_scatter_finalize(ta, tc, finalize_slice)
    assert labels.dtype == torch.int32 and labels.shape == (acc.shape[0],)
    np.save(out + "_labels%d.npy" % rank, labels.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_reduce_scatter_finalize_equals_single_rank_labels(tmp_path, world):
    """The product exchange (dist.reduce_scatter_rows + reduce_scatter_finalize: reduce_scatter_tensor,
    slice-wise finalize, all_gather_into_tensor) == one-rank labels.  cfg1 has 13,468 texels: world 2
    and 4 divide it (no padding copy), world 3 does not (padded last slice)."""
    out = str(tmp_path / "rs")
    mp.spawn(_rs_worker, args=(world, _free_port(), "mul", out), nprocs=world, join=True)
    import oracle as O

    z, probs = _scene()
    acc1, cnt1 = _fold(z, probs, range(len(z["cams"])), "mul")
    rows, unobs = O.finalize(acc1, cnt1, "mul")
    ref = O.texel_argmax(rows, unobs)
    k = (len(cnt1) + world - 1) // world
    for r in range(world):
        lo, hi = np.load(out + "_bounds%d.npy" % r)
        assert (lo, hi) == (min(len(cnt1), r * k), min(len(cnt1), (r + 1) * k))
        sl = np.load(out + "_slice%d.npy" % r)
        np.testing.assert_allclose(sl[:, :-1], acc1[lo:hi], rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(sl[:, -1], cnt1[lo:hi])
        got = np.load(out + "_labels%d.npy" % r)
        decided = np.ones(len(ref), bool)
        top2 = np.sort(rows, axis=1)[:, -2:]
        decided &= (top2[:, 1] - top2[:, 0]) > 1e-9
        np.testing.assert_array_equal(got[decided | unobs], ref[decided | unobs])

"""Frame sharding and the single accumulator exchange for multi-GPU fusion.

All three aggregation rules are sums (fusion.py:5-17: sum of w*p, masked sum,
sum of w*log p) and the observation counts are sums too, so P ranks that
each fold a disjoint block of frames into a private accumulator reproduce the
one-rank texture with ONE sum all-reduce of (accumulator, counts) before
finalize.  Weights (images_iid / blend) are per frame and stay
rank-local.  After the exchange every rank holds the fused texture and can
re-render its own frames with no further communication.

Backend: NCCL over NVLink/NVSwitch on GPUs (torch.distributed "nccl"); the
same code runs on "gloo" with CPU tensors, which is how the host logic is
tested without GPUs (tests/test_dist_gloo.py).
"""

import os

import torch
import torch.distributed as dist


def world():
    """(rank, world_size) of the default group, (0, 1) when not distributed."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_bounds(num_frames, rank, world_size):
    """Contiguous block [lo, hi) of frames for ``rank`` (consecutive frames
    see overlapping texels, which keeps a rank's accumulator traffic local)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank %r / world size %r" % (rank, world_size))
    lo = num_frames * rank // world_size
    hi = num_frames * (rank + 1) // world_size
    return lo, hi


def shard_frames(frames, rank=None, world_size=None):
    """This rank's block of a frame sequence."""
    if rank is None or world_size is None:
        rank, world_size = world()
    lo, hi = shard_bounds(len(frames), rank, world_size)
    return frames[lo:hi]


def allreduce_sum_(tensors, group=None):
    """In-place SUM all-reduce of each tensor (accumulator rows, counts)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return tensors
    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return tensors


def _supports_reduce_scatter(group):
    return dist.get_backend(group) == "nccl"


def reduce_scatter_finalize(accum, counts, finalize_slice, group=None):
    """Exchange + finalize with the work split over ranks (fused variant).

    Instead of every rank receiving the whole summed accumulator, texel rows
    are cut into P contiguous slices: a sum reduce-scatter gives rank r the
    summed rows [r*k, (r+1)*k) (k = ceil(n/P)), the rank finalizes only that
    slice (``finalize_slice(acc_slice, counts_slice) -> int32 labels``) and
    the int32 labels are all-gathered (4 B per texel instead of the 4c-byte
    rows).  Returns the (n,) int32 labels, identical on every rank.

    NCCL runs reduce-scatter; on backends without it (gloo, used by the CPU
    tests) the rows are all-reduced and sliced locally, with the same result.
    """
    rank, world_size = (dist.get_rank(group), dist.get_world_size(group)) if (
        dist.is_available() and dist.is_initialized()) else (0, 1)
    n = int(accum.shape[0])
    if world_size == 1:
        return finalize_slice(accum, counts)
    k = (n + world_size - 1) // world_size
    lo, hi = min(n, rank * k), min(n, (rank + 1) * k)
    if _supports_reduce_scatter(group):
        acc_pad = torch.zeros((k * world_size,) + tuple(accum.shape[1:]), dtype=accum.dtype, device=accum.device)
        acc_pad[:n] = accum
        cnt_pad = torch.zeros(k * world_size, dtype=counts.dtype, device=counts.device)
        cnt_pad[:n] = counts
        acc_mine = torch.empty((k,) + tuple(accum.shape[1:]), dtype=accum.dtype, device=accum.device)
        cnt_mine = torch.empty(k, dtype=counts.dtype, device=counts.device)
        dist.reduce_scatter_tensor(acc_mine, acc_pad, op=dist.ReduceOp.SUM, group=group)
        dist.reduce_scatter_tensor(cnt_mine, cnt_pad, op=dist.ReduceOp.SUM, group=group)
        acc_mine, cnt_mine = acc_mine[: hi - lo], cnt_mine[: hi - lo]
    else:
        acc_all, cnt_all = accum.clone(), counts.clone()
        dist.all_reduce(acc_all, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(cnt_all, op=dist.ReduceOp.SUM, group=group)
        acc_mine, cnt_mine = acc_all[lo:hi], cnt_all[lo:hi]
    mine = torch.full((k,), -1, dtype=torch.int32, device=accum.device)
    if hi > lo:
        mine[: hi - lo] = finalize_slice(acc_mine.contiguous(), cnt_mine.contiguous())
    parts = [torch.empty_like(mine) for _ in range(world_size)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat(parts)[:n]


def init_from_env(backend=None):
    """Initialise the default process group from torchrun's environment
    (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT); returns (rank, world, local_rank)."""
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world_size > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend, init_method="env://")
    return rank, world_size, local

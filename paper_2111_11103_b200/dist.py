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

"""Frame sharding and the single accumulator exchange for multi-GPU fusion.

All three aggregation rules are sums (fusion.py:5-17: sum of w*p, masked sum,
sum of w*log p) and the observation counts are sums too, so P ranks that
each fold a disjoint block of frames into a private accumulator reproduce the
one-rank texture with ONE sum all-reduce of (accumulator, counts) before
finalize.  Weights (images_iid / blend) are per frame and stay
rank-local.  After the exchange every rank holds the fused texture and can
re-render its own frames with no further communication.

Backend: NCCL over NVLink/NVSwitch on GPUs (torch.distributed "nccl"); the
same calls (reduce_scatter_tensor, all_gather_into_tensor, all_reduce) run on
"gloo" with CPU tensors, which is how the exchange is tested without GPUs
(tests/test_dist_gloo.py, world sizes 2 and 3: with and without padding).
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


def _padded(t, rows):
    """``t`` itself when it already has ``rows`` rows, else a zero-padded copy
    (reduce-scatter needs equal slices; n % P == 0 at every BASELINE config)."""
    if int(t.shape[0]) == rows:
        return t
    pad = torch.zeros((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: int(t.shape[0])] = t
    return pad


def reduce_scatter_rows(tensors, group=None):
    """Sum reduce-scatter of each tensor's leading (texel-row) dimension.

    Rank r receives the summed rows [r*k, (r+1)*k) of every tensor, k =
    ceil(n/P); rows past n are padding.  One ``reduce_scatter_tensor`` per
    tensor (NCCL ring / NVLS on the GPU box, gloo's implementation on the
    CPU tests: the same call either way).  Returns (slices, (lo, hi))."""
    rank, world_size = dist.get_rank(group), dist.get_world_size(group)
    n = int(tensors[0].shape[0])
    k = (n + world_size - 1) // world_size
    lo, hi = min(n, rank * k), min(n, (rank + 1) * k)
    out = []
    for t in tensors:
        src = _padded(t if t.is_contiguous() else t.contiguous(), k * world_size)
        mine = torch.empty((k,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.reduce_scatter_tensor(mine, src, op=dist.ReduceOp.SUM, group=group)
        out.append(mine[: hi - lo])
    return out, (lo, hi)


def reduce_scatter_finalize(accum, counts, finalize_slice, group=None, exchange_single=False):
    """Exchange + finalize with the work split over ranks (fused variant).

    Instead of every rank receiving the whole summed accumulator, texel rows
    are cut into P contiguous slices: a sum reduce-scatter gives rank r the
    summed rows [r*k, (r+1)*k) (k = ceil(n/P)), the rank finalizes only that
    slice (``finalize_slice(acc_slice, counts_slice) -> int32 labels``) and
    the int32 labels are all-gathered (4 B per texel instead of the 4c-byte
    rows).  Returns the (n,) int32 labels, identical on every rank.
    ``exchange_single`` runs the collectives even in a one-rank group (tests drive
    the NCCL calls on a single GPU with it).
    """
    initialized = dist.is_available() and dist.is_initialized()
    world_size = dist.get_world_size(group) if initialized else 1
    n = int(accum.shape[0])
    if world_size == 1 and not (exchange_single and initialized):
        return finalize_slice(accum, counts)
    k = (n + world_size - 1) // world_size
    (acc_mine, cnt_mine), (lo, hi) = reduce_scatter_rows([accum, counts], group)
    mine = torch.full((k,), -1, dtype=torch.int32, device=accum.device)
    if hi > lo:
        mine[: hi - lo] = finalize_slice(acc_mine.contiguous(), cnt_mine.contiguous())
    labels = torch.empty((k * world_size,), dtype=torch.int32, device=accum.device)
    dist.all_gather_into_tensor(labels, mine, group=group)
    return labels[:n]


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

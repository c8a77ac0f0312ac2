"""MeshAnnotation-style fusion: ``add(probs, camera)`` / ``get()`` / ``render(camera)``.

The batched, device-resident front end of the hot path (BASELINE north star):
for each batch of up to ``max_batch`` frames of one size it issues the
stream-ordered launches of tfb_rasterize (cluster cull, setup + tile
binning, tile raster with the per-frame texel hit counts fused into its
epilogue), one tfb_fuse scatter-add and the hit-counter reset, and never
synchronizes with the host.  Host inputs are copied on a separate stream
into double-buffered device staging, overlapping the previous batch's
kernels.  ``get()`` finalizes once (tfb_finalize) and returns the per-texel
rows; ``render`` rasterizes the requested cameras and gathers labels
(tfb_render).  Multi-GPU: each rank adds its own frames, then
``finalize_distributed()`` (reduce-scatter, slice finalize, label
all-gather) or ``allreduce()`` (then ``get()``).

Per-frame calls run at batched speed: ``add(probs, camera)`` (and the
session's ``add_frame``, bindings/__init__.py:85-115) only queue the frame;
the queue is folded as one batch when it reaches ``max_batch`` frames, when
the frame size changes, and before anything reads the texture (``get``,
``labels``, ``render``, ``texture``, checkpoints, the exchange).  Host
inputs are copied to the device when queued (so the caller may reuse its
array at once, as with the reference's copy at bindings/__init__.py:101);
device float32 tensors are used in place and must not be modified before
the queue is folded -- an in-place write is detected through the tensor's
version counter and raises instead of fusing changed data.

It is a thin layer over the same ProbabilityTexture the reference-compatible
functions use (fusion.py / session.py), so textures and results interchange.
"""

import os
import weakref

import numpy as np
import torch

from . import _native as N
from .device import scene_for
from .errors import DataError
from .fusion import init_texture, parse_weight_mode
from .geometry import pack_camera, uniform_layout
from .renderback import render_labels_device

MAX_BATCH_CAP = 256  # tfb_fuse carries at most 256 frames per launch


def _cams_array(cameras):
    if isinstance(cameras, torch.Tensor):
        return cameras.detach().to(torch.float64).reshape(-1, 16)
    if isinstance(cameras, np.ndarray) and cameras.ndim == 2 and cameras.shape[1] == 16:
        return torch.as_tensor(np.ascontiguousarray(cameras, dtype=np.float64))
    if not isinstance(cameras, (list, tuple)):
        cameras = [cameras]
    return torch.as_tensor(np.stack([pack_camera(c) for c in cameras]))


def _sizes(cameras, width, height):
    if width is not None and height is not None:
        return int(width), int(height)
    cam0 = cameras[0] if isinstance(cameras, (list, tuple)) else cameras
    return int(cam0.width), int(cam0.height)


def _device_ready(p, device):
    """True for tensors the scatter-add can read in place."""
    return (isinstance(p, torch.Tensor) and p.is_cuda and p.device == device and p.dtype == torch.float32
            and p.is_contiguous() and p.data_ptr() % 16 == 0)


class _Pending:
    """A queued frame: device probabilities, packed camera, and what to report back."""

    __slots__ = ("probs", "cam", "version", "ids", "ready", "fallback_key")

    def __init__(self, probs, cam, version, ids=None, ready=None, fallback_key=None):
        self.probs = probs
        self.cam = cam
        self.version = version
        self.ids = ids
        self.ready = ready
        self.fallback_key = fallback_key


class FrameCount:
    """Covered pixels of one queued frame (the int add_frame returns,
    bindings/__init__.py:113), computed only when read -- from the frame's lazy
    IdImage, so reading it neither folds the queue nor costs the unread ones."""

    __slots__ = ("_ids", "_scene", "_v")

    def __init__(self, ids, scene):
        self._ids = ids
        self._scene = scene
        self._v = None

    def __int__(self):
        if self._v is None:
            self._v = int((self._ids.rows_on(self._scene) >= 0).sum().item())
            self._ids = self._scene = None
        return self._v

    __index__ = __int__

    def __eq__(self, o):
        return int(self) == int(o)

    def __ne__(self, o):
        return int(self) != int(o)

    def __lt__(self, o):
        return int(self) < o

    def __le__(self, o):
        return int(self) <= o

    def __gt__(self, o):
        return int(self) > o

    def __ge__(self, o):
        return int(self) >= o

    def __hash__(self):
        return hash(int(self))

    def __add__(self, o):
        return int(self) + o

    __radd__ = __add__

    def __sub__(self, o):
        return int(self) - o

    def __rsub__(self, o):
        return o - int(self)

    def __repr__(self):
        return repr(int(self))


class _PinnedStager:
    """Pageable host maps -> device through a ring of pinned bounce buffers.

    A copy from pageable memory goes through the driver's own staging at one
    host thread's memcpy speed (~11 GB/s measured, a fifth of the PCIe link).
    Here a few host threads copy the maps into pinned slots (NumPy's copy
    releases the GIL) while the DMA engine drains earlier slots, so host copy,
    H2D and the kernels all overlap."""

    def __init__(self, slots=8, threads=None):
        import os
        from concurrent.futures import ThreadPoolExecutor

        # 8 threads measured best on a 16-core host (876 vs 832 frames/s with 16 at cfg2);
        # with several ranks per host (LOCAL_WORLD_SIZE, set by torchrun) they share the cores
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 2
        local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1))
        n = threads or int(os.environ.get("TFB_STAGE_THREADS", "0")) or max(1, min(8, cores // local))
        self.pool = ThreadPoolExecutor(max_workers=n, thread_name_prefix="tfb-stage")
        self.nthreads = n
        self.nslots = slots
        self.slots = []  # (pinned float32 tensor (numel,), event of the H2D that last read it)
        self.size = 0
        self.next = 0

    def _ensure(self, numel):
        if numel > self.size:
            self.slots = [[torch.empty(numel, dtype=torch.float32).pin_memory(), None] for _ in range(self.nslots)]
            self.size = numel

    def upload(self, pairs, stream):
        """pairs: [(host array-like, device float32 destination)], copied in order on ``stream``."""
        self._ensure(max(int(d.numel()) for _, d in pairs))
        pending = []

        def fill(host, src):
            np.copyto(host, src, casting="unsafe")

        for src, dst in pairs:
            k = self.next
            self.next = (k + 1) % self.nslots
            slot = self.slots[k]
            if slot[1] is not None:
                slot[1].synchronize()  # the DMA that last read this slot is done
            host = slot[0][: dst.numel()].numpy().reshape(dst.shape)
            src = np.asarray(src)
            # one map is split over the threads by rows, so even a single frame copies at
            # several threads' bandwidth
            step = max(1, -(-host.shape[0] // self.nthreads))
            futs = [self.pool.submit(fill, host[r:r + step], src[r:r + step]) for r in range(0, host.shape[0], step)]
            pending.append((futs, slot, dst))
            if len(pending) == self.nslots:
                self._drain(pending.pop(0), stream)
        for item in pending:
            self._drain(item, stream)

    @staticmethod
    def _drain(item, stream):
        futs, slot, dst = item
        for f in futs:
            f.result()
        with torch.cuda.stream(stream):
            dst.copy_(slot[0][: dst.numel()].view(dst.shape), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        slot[1] = ev


class FallbackMap(dict):
    """key -> (H*W,) int32 device network argmax of a folded frame; entries are
    stored as (batch buffer, index) and viewed on access (no per-frame views).
    ``reserve`` pre-sizes one arena per frame size (a session knows its
    trajectory), so folds take rows from it instead of allocating per batch."""

    def __init__(self):
        super().__init__()
        self._arena = {}  # (W, H) -> [tensor (n, H*W) int32 or None, capacity, next free row]

    def reserve(self, size, nframes):
        self._arena[size] = [None, int(nframes), 0]

    def rows_for(self, size, b, device):
        """(b, H*W) int32 device rows for the network argmax of b frames."""
        a = self._arena.get(size)
        hw = size[0] * size[1]
        if a is not None and a[2] + b <= a[1]:
            if a[0] is None:
                a[0] = torch.empty((a[1], hw), dtype=torch.int32, device=device)
            out = a[0][a[2]:a[2] + b]
            a[2] += b
            return out
        return torch.empty((b, hw), dtype=torch.int32, device=device)

    def __getitem__(self, key):
        buf, k = dict.__getitem__(self, key)
        return buf[k]

    def get(self, key, default=None):
        return self[key] if key in self else default


class MeshAnnotation:
    """Fuse per-frame class probabilities onto a mesh's texels on the GPU."""

    def __init__(self, mesh, layout=None, num_classes=None, aggregator="mul", weight_mode="images_iid",
                 accum_dtype="float32", max_batch=None, device=None, memory_budget=None, overlap=False,
                 fuse_ctas_per_sm=None, texture=None, order_items=None, split_raster=None):
        if texture is None and num_classes is None:
            raise ValueError("num_classes is required")
        self.mesh = mesh
        self.layout = layout if layout is not None else (texture.layout if texture is not None
                                                          else uniform_layout(mesh, 1))
        self.weight_mode, self.alpha = parse_weight_mode(weight_mode)
        if texture is None:
            budget = memory_budget if memory_budget is not None else float("inf")
            texture = init_texture(self.layout, int(num_classes), aggregator, budget, accum_dtype, device)
        self._tex = texture
        self.num_classes = int(texture.num_classes)
        self.scene = scene_for(mesh, self.layout, texture.device)
        self.device = self.scene.device
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        # None: sized per frame size from the free device memory (_batch_for)
        self.max_batch = None if max_batch is None else max(1, min(int(max_batch), MAX_BATCH_CAP))
        self._auto_batch = {}
        self._staging = [None, None]  # device staging for host inputs (double-buffered)
        self._stage_free = [None, None]
        self._stage_slot = 0
        self._copy_stream = None
        self._stager = None  # pinned bounce ring for pageable host maps (created on first use)
        self.frames_added = 0
        self._pending = []
        self._pending_size = None
        self._cam_ring = None
        # row-block item order for the scatter-add (tfb_fuse_order): None = when the
        # accumulator exceeds half the L2 (configs[3]), True / False to force it
        self.order_items = order_items
        texture._flush_hook = weakref.WeakMethod(self.flush)
        # Overlap mode: batch k+1 is rasterized on a side stream while batch k
        # is scatter-added on the caller's stream (double-buffered row / hit
        # images); the scatter kernel is capped at fuse_ctas_per_sm resident
        # CTAs so rasterizer CTAs can share the SMs.
        self.overlap = bool(overlap)
        self._side = torch.cuda.Stream(self.device) if self.overlap else None
        self._free = [None, None]
        # Split mode: the rasterizer's first phase (cull, record setup, tile binning: latency
        # bound, little issue) of batch k+1 runs on a side stream under batch k's scatter-add
        # (bandwidth bound); its second phase (the tile kernels) stays in stream order.  One
        # workspace and one row / hit image suffice (tfb_rasterize_phases).
        if split_raster is None:  # opt-in (TFB_SPLIT_RASTER=1): +1.5-2 % frames/s at cfg2, but the
            # scatter-add then shares the GPU and its own roofline reads 0.87 instead of 0.97
            split_raster = os.environ.get("TFB_SPLIT_RASTER", "0") == "1"
        self.split_raster = bool(split_raster) and not self.overlap
        self._split_side = (torch.cuda.Stream(self.device, priority=int(os.environ.get("TFB_SPLIT_PRIO", "0")))
                            if self.split_raster else None)
        if fuse_ctas_per_sm is None:
            fuse_ctas_per_sm = 2 if self.overlap else 0
        N.call("tfb_set_option", 1, int(fuse_ctas_per_sm))
        # optional list receiving (frames, ev_raster_start, ev_raster_end, ev_fuse_start, ev_fuse_end)
        self.profile = None

    @property
    def texture(self):
        """The fused ProbabilityTexture (queued frames are folded first)."""
        self.flush()
        return self._tex

    @staticmethod
    def _event(stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _batch_for(self, W, H):
        """Frames per batch: max_batch, or what a quarter of the free device
        memory holds (raster workspace + row image + hit counts + host staging)."""
        if self.max_batch is not None:
            return self.max_batch
        b = self._auto_batch.get((W, H))
        if b is None:
            lib = N.load()
            nv, m = int(self.scene.struct.num_vertices), self.scene.num_triangles
            ws1 = lib.tfb_raster_workspace_bytes(nv, m, W, H, 1, 0)
            ws2 = lib.tfb_raster_workspace_bytes(nv, m, W, H, 2, 0)
            per = (ws2 - ws1) + W * H * 4 * (2 + self.num_classes) + max(self._tex.total_texels, 1) * 4
            # what is free plus what the caching allocator holds unused (blocks of earlier
            # jobs count as used to the driver but are ours to reuse)
            free, _total = torch.cuda.mem_get_info(self.device)
            cached = torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
            b = int(max(1, min(MAX_BATCH_CAP, ((free + cached) // 4 - ws1) // max(per, 1))))
            self._auto_batch[(W, H)] = b
        return b

    def reset(self):
        """Zero the accumulator and counts for a new fusion job (same layout);
        frames still queued belong to the old job and are dropped."""
        self._pending = []
        self._pending_size = None
        tex = self._tex
        tex._accum.zero_()
        tex._counts.zero_()
        tex.finalized = False
        tex._rows = tex._unobs = tex._labels = None
        tex._h_accum = tex._h_counts = tex._h_rows = tex._h_unobs = None
        self.frames_added = 0

    # -- checkpoint / resume (the accumulator is a sum monoid) --------------
    CHECKPOINT_VERSION = 1

    def save_checkpoint(self, path):
        """Write the un-finalized accumulation state (accumulator rows, counts,
        frames added and what they must match) to ``path`` (.npz).  A job
        resumed from it with load_checkpoint() and fed the remaining frames
        ends with the same fused result (sums, up to float rounding order)."""
        tex = self.texture
        if tex.finalized:
            raise RuntimeError("texture is already finalized; checkpoint before labels()/render()")
        tex._push_host()
        torch.cuda.synchronize(self.device)
        np.savez(path, version=np.int64(self.CHECKPOINT_VERSION),
                 accum=tex.accum_values().cpu().numpy(), counts=tex._counts.cpu().numpy(),
                 frames_added=np.int64(self.frames_added), num_classes=np.int64(self.num_classes),
                 aggregator=np.array(tex.aggregator), weight_mode=np.array(self.weight_mode),
                 alpha=np.float64(self.alpha or 0.0), total_texels=np.int64(tex.total_texels),
                 accum_dtype=np.array(str(tex.dtype).replace("torch.", "")),
                 steps=self.layout.steps, offsets=self.layout.offsets)

    def load_checkpoint(self, path):
        """Resume from save_checkpoint(): the accumulator and counts are
        replaced by the saved ones.  The checkpoint must come from the same
        layout, class count, aggregator and weight mode (DataError otherwise);
        per-rank checkpoints of a sharded job can be loaded on their ranks and
        reduced as usual."""
        tex = self._tex
        with np.load(path, allow_pickle=False) as z:
            if int(z["version"]) != self.CHECKPOINT_VERSION:
                raise DataError("checkpoint version %d is not supported" % int(z["version"]))
            want = {"num_classes": self.num_classes, "total_texels": tex.total_texels}
            for key, val in want.items():
                if int(z[key]) != int(val):
                    raise DataError("checkpoint %s %d does not match %d" % (key, int(z[key]), int(val)))
            if str(z["aggregator"]) != tex.aggregator or str(z["weight_mode"]) != self.weight_mode or \
                    float(z["alpha"]) != float(self.alpha or 0.0):
                raise DataError("checkpoint aggregator / weight mode (%s, %s) do not match (%s, %s)" % (
                    str(z["aggregator"]), str(z["weight_mode"]), tex.aggregator, self.weight_mode))
            if not (np.array_equal(z["steps"], self.layout.steps) and np.array_equal(z["offsets"], self.layout.offsets)):
                raise DataError("checkpoint texel layout does not match")
            accum, counts = z["accum"], z["counts"]
            if accum.shape != (tex.total_texels, self.num_classes) or counts.shape != (tex.total_texels,):
                raise DataError("checkpoint arrays have the wrong shape")
            self.reset()
            tex._accum[:, : self.num_classes].copy_(tex.accum_from_values(accum))
            tex._counts.copy_(torch.as_tensor(counts).to(self.device, tex._counts.dtype))
            self.frames_added = int(z["frames_added"])

    # -- accumulation ------------------------------------------------------------------
    def _probs_batch(self, probs, b, H, W, cur, cap):
        """Per-frame device pointers for b frames.  Contiguous float32 device
        tensors are used in place; other device tensors (float16, permuted,
        unaligned) are converted on the caller's stream ``cur``, where they were
        produced; host arrays / tensors are copied into one of two device
        staging buffers on a copy stream, so the copy of batch k+1 overlaps the
        kernels of batch k.  Returns (pointers, keep-alive list, copy-done event
        or None, staging slot)."""
        c = self.num_classes
        if isinstance(probs, (list, tuple)):
            items = list(probs)
        else:
            items = [probs[i] for i in range(b)] if probs.ndim == 4 else [probs]
        for p in items:
            if tuple(p.shape) != (H, W, c):
                raise DataError("probability array shape %s does not match expected %s"
                                % (tuple(p.shape), (H, W, c)))
        for i, p in enumerate(items):
            if isinstance(p, torch.Tensor) and p.is_cuda and not _device_ready(p, self.device):
                with torch.cuda.stream(cur):
                    q = p.detach().to(device=self.device, dtype=torch.float32).contiguous()
                    if q.data_ptr() % 16 or q.data_ptr() == p.data_ptr():
                        q = q.clone()
                items[i] = q  # made on cur, read on cur: no cross-stream lifetime to track
        need_stage = [i for i, p in enumerate(items) if not (isinstance(p, torch.Tensor) and p.is_cuda)]
        ready, slot = None, None
        if need_stage:
            shape = (cap, H, W, c)
            slot = self._stage_slot
            self._stage_slot ^= 1
            if self._staging[slot] is None or tuple(self._staging[slot].shape) != shape:
                self._staging[slot] = torch.empty(shape, dtype=torch.float32, device=self.device)
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(self.device)
            cs = self._copy_stream
            if self._stage_free[slot] is not None:
                cs.wait_event(self._stage_free[slot])  # the scatter that last read this buffer is done
            pageable = []
            with torch.cuda.stream(cs):
                for k, i in enumerate(need_stage):
                    p, dst = items[i], self._staging[slot][k]
                    if isinstance(p, torch.Tensor) and p.is_pinned():
                        dst.copy_(p, non_blocking=True)
                    else:
                        pageable.append((p.numpy() if isinstance(p, torch.Tensor) else p, dst))
                    items[i] = dst
            if pageable:
                if self._stager is None:
                    self._stager = _PinnedStager()
                self._stager.upload(pageable, cs)
            ready = torch.cuda.Event()
            ready.record(cs)
        return [p.data_ptr() for p in items], items, ready, slot

    def add_batch(self, probs, cameras, width=None, height=None, fallback_out=None, stream=None):
        """Fold B frames: probs (B, H, W, c) tensor/array or a list of (H, W, c);
        cameras a list of CameraFrame or a (B, 16) camera array/tensor.
        fallback_out (optional (B, H*W) int32 device tensor) receives each
        frame's network argmax."""
        self.flush()
        with torch.cuda.device(self.device):
            W, H = _sizes(cameras, width, height)
            cur = stream if stream is not None else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(cur):
                cams_all = _cams_array(cameras).to(self.device, non_blocking=True)
            self._fold(probs, cams_all, W, H, fallback_out, cur)

    def _fold(self, probs, cams_all, W, H, fallback_out, cur, ready=()):
        """The batched pipeline over B frames with device cameras ``cams_all``."""
        tex = self._tex
        if tex.finalized:
            raise RuntimeError("texture is already finalized")
        B = int(cams_all.shape[0])
        hw = H * W
        tex._push_host()
        for ev in ready:
            cur.wait_event(ev)
        needs_hits = self.weight_mode != "pixels_iid"
        nslots = 2 if self.overlap else 1
        mb = self._batch_for(W, H) if B > 1 else 1
        mb = min(mb, B) if self.max_batch is None else mb
        rows_all = self.scene.buffer("rows", (nslots, mb, hw), torch.int32)
        hits_all = (self.scene.buffer("hits2", (nslots, mb, max(tex.total_texels, 1)), torch.int32, zero=True)
                    if needs_hits else None)
        side = self._side if self.overlap else cur
        if self.overlap:
            side.wait_stream(cur)  # cameras and anything queued before this call
            cams_all.record_stream(side)
        split = self.split_raster and B > mb
        if split:
            sside = self._split_side
            sside.wait_stream(cur)
            cams_all.record_stream(sside)
            self.scene.workspace(W, H, mb)  # sized once: never regrown while the side stream uses it
            setup_done = None
        for i, b0 in enumerate(range(0, B, mb)):
            b = min(mb, B - b0)
            slot = i % nslots
            chunk = probs[b0:b0 + b]
            ptrs, keep, copied, sslot = self._probs_batch(chunk, b, H, W, cur, mb)
            rows = rows_all[slot, :b]
            hits = hits_all[slot, :b] if needs_hits else None
            if self.overlap and self._free[slot] is not None:
                side.wait_event(self._free[slot])  # the scatter that last read this slot is done
            prof = self.profile
            r0 = self._event(side) if prof is not None else None
            if split:
                if setup_done is None:
                    self.scene.rasterize(cams_all[b0:b0 + b], W, H, rows, hits=hits, stream=cur, phases=1)
                else:
                    cur.wait_event(setup_done)
                self.scene.rasterize(cams_all[b0:b0 + b], W, H, rows, hits=hits, stream=cur, phases=2)
                drawn = torch.cuda.Event()
                drawn.record(cur)  # this batch's tile kernels are done with the workspace
            else:
                self.scene.rasterize(cams_all[b0:b0 + b], W, H, rows, hits=hits, stream=side)
            r1 = self._event(side) if prof is not None else None
            if self.overlap:
                ev = torch.cuda.Event()
                ev.record(side)
                cur.wait_event(ev)
            if copied is not None:
                cur.wait_event(copied)
            f0 = self._event(cur) if prof is not None else None
            parr, _k = N.ptr_array(ptrs)
            fb = fallback_out[b0:b0 + b] if fallback_out is not None else None
            order, n_order = self._item_order(rows, hw, b, fb, cur)
            N.call("tfb_fuse_ordered", N.ptr(rows), hw, b, parr, self.num_classes, N.ptr(hits), None,
                   tex.total_texels, N.AGG_IDS[tex.aggregator], N.WMODE_IDS[self.weight_mode],
                   float(self.alpha or 0.0), N.ptr(tex._accum), tex.accum_kind, tex.stride, N.ptr(tex._counts),
                   N.ptr(fb), N.ptr(order), N.ptr(n_order), N.stream_handle(cur))
            if split and b0 + mb < B:
                # the next batch's first phase under this batch's scatter-add, enqueued after it
                # so the scatter-add's persistent CTAs are placed first
                nb0, nb = b0 + mb, min(mb, B - b0 - mb)
                sside.wait_event(drawn)
                with torch.cuda.stream(sside):
                    self.scene.rasterize(cams_all[nb0:nb0 + nb], W, H, rows[:nb], stream=sside, phases=1)
                setup_done = torch.cuda.Event()
                setup_done.record(sside)
            if prof is not None:
                prof.append((b, r0, r1, f0, self._event(cur)))
            if sslot is not None:
                ev = torch.cuda.Event()
                ev.record(cur)
                self._stage_free[sslot] = ev
            if needs_hits:
                if tex.total_texels <= 4 * hw:  # a dense memset is cheaper than the scattered reset
                    with torch.cuda.stream(cur):
                        hits.zero_()
                else:
                    N.call("tfb_clear_hits", N.ptr(rows), hw, b, tex.total_texels, N.ptr(hits),
                           N.stream_handle(cur))
            if self.overlap:
                ev = torch.cuda.Event()
                ev.record(cur)
                self._free[slot] = ev
            del keep
        tex._h_accum = tex._h_counts = None
        self.frames_added += B

    ORDER_SHIFT = 10  # item-order key = accumulator row block of 1024 rows

    def _use_order(self):
        """Auto: the float32 fast path (the kernel that walks an order) with 16-byte class
        quads (c % 4 == 0), when the accumulator exceeds half the L2.  Measured at
        configs[3] (1.73 GB): scatter-add 32.9 -> 15.3 us/frame.  The c % 4 != 0 kernel is
        issue-bound rather than bound by accumulator traffic, and the order's extra work
        makes it slower (configs[4], c = 19: 47.0 -> 55.2 us/frame), so it walks
        frame-major."""
        if self.order_items is not None:
            return bool(self.order_items)
        tex = self._tex
        if tex.accum_kind != 0 or self.num_classes % 4:
            return False
        l2 = torch.cuda.get_device_properties(self.device).L2_cache_size
        return tex.total_texels * tex.stride * 4 > l2 // 2

    def _item_order(self, rows, hw, b, fb, cur):
        """(order, count) device buffers from tfb_fuse_order, or (None, None)."""
        if fb is not None or not self._use_order():
            return None, None
        tex = self._tex
        lib = N.load()
        nbytes = lib.tfb_fuse_order_workspace_bytes(hw, b, tex.total_texels, self.ORDER_SHIFT)
        ws = self.scene.buffer("order_ws", (nbytes,), torch.uint8)
        order = self.scene.buffer("order", (b * ((hw + 31) // 32),), torch.int32)
        n_order = self.scene.buffer("order_n", (1,), torch.int32)
        N.call("tfb_fuse_order", N.ptr(rows), hw, b, tex.total_texels, self.ORDER_SHIFT, N.ptr(ws), nbytes,
               N.ptr(order), N.ptr(n_order), N.stream_handle(cur))
        return order, n_order

    # -- per-frame queue ---------------------------------------------------------------
    def _stage_one(self, probs, H, W, cur):
        """Device float32 copy (or the tensor itself) of one frame's probabilities, and
        the version to check at fold time (None when the copy is ours)."""
        c = self.num_classes
        shape = tuple(probs.shape) if hasattr(probs, "shape") else np.shape(probs)
        if shape != (H, W, c):
            raise DataError("probability array shape %s does not match expected %s" % (shape, (H, W, c)))
        if _device_ready(probs, self.device):
            return probs.detach(), probs._version, None
        if isinstance(probs, torch.Tensor) and probs.is_cuda:
            with torch.cuda.stream(cur):
                q = probs.detach().to(device=self.device, dtype=torch.float32).contiguous()
                if q.data_ptr() % 16 or q.data_ptr() == probs.data_ptr():
                    q = q.clone()
            return q, None, None
        # host input: copied now (the caller may reuse its array once this returns), on the
        # copy stream; pageable memory through the pinned bounce ring
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        cs = self._copy_stream
        with torch.cuda.stream(cs):
            q = torch.empty((H, W, c), dtype=torch.float32, device=self.device)
        if isinstance(probs, torch.Tensor) and probs.is_pinned():
            with torch.cuda.stream(cs):
                q.copy_(probs.detach(), non_blocking=True)
        else:
            if self._stager is None:
                self._stager = _PinnedStager()
            self._stager.upload([(probs.detach().numpy() if isinstance(probs, torch.Tensor) else probs, q)], cs)
        ev = torch.cuda.Event()
        ev.record(cs)
        q.record_stream(cur)
        return q, None, ev

    def _enqueue(self, probs, camera, ids=None, fallback_key=None, want_count=False):
        tex = self._tex
        if tex.finalized:
            raise RuntimeError("texture is already finalized")
        intr = camera.intrinsics
        W, H = int(intr.width), int(intr.height)
        if self._pending and self._pending_size != (W, H):
            self.flush()
        src = getattr(ids, "_source", None)
        cam = src[1] if src is not None else pack_camera(camera)
        if (type(probs) is torch.Tensor and probs.is_cuda and probs.dtype is torch.float32
                and probs.get_device() == self._dev_index and probs.is_contiguous() and not probs.data_ptr() & 15):
            if probs.shape != (H, W, self.num_classes):
                raise DataError("probability array shape %s does not match expected %s"
                                % (tuple(probs.shape), (H, W, self.num_classes)))
            item = _Pending(probs, cam, probs._version, ids, None, fallback_key)
        else:
            with torch.cuda.device(self.device):
                p, version, ready = self._stage_one(probs, H, W, torch.cuda.current_stream(self.device))
            item = _Pending(p, cam, version, ids, ready, fallback_key)
        self._pending.append(item)
        self._pending_size = (W, H)
        if len(self._pending) >= self._batch_for(W, H):
            self.flush()
        return FrameCount(ids, self.scene) if want_count else None

    def add(self, probs, camera, **kw):
        """Queue one (H, W, c) probability map seen from ``camera``; it is folded
        with the frames queued next to it as one batch (see the module doc).
        With keyword arguments (width/height/fallback_out/stream) the frame is
        folded at once through add_batch."""
        if kw or isinstance(camera, (list, tuple)):
            cams = list(camera) if isinstance(camera, (list, tuple)) else [camera]
            self.add_batch([probs], cams, **kw)
            return
        self._enqueue(probs, camera)

    # session hooks (session.py): results of queued frames ------------------------------
    fallbacks = None  # FallbackMap key -> (H*W,) int32 device network argmax, when a session asks for it

    def flush(self):
        """Fold the queued frames (one batched pass per max_batch frames)."""
        pend = self._pending
        if not pend:
            return
        self._pending = []
        W, H = self._pending_size
        self._pending_size = None
        for k, it in enumerate(pend):
            if it.version is not None and it.probs._version != it.version:
                raise RuntimeError("the probability tensor of queued frame %d was modified in place before the "
                                   "queue was folded; pass a copy, or call flush() before reusing the buffer" % k)
        hw = H * W
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            # frames whose IdImage came from some other rasterization (a hook returning a
            # prepared IdImage) fold with their own row image, one at a time
            own = [it for it in pend if it.ids is None or self._ids_from_camera(it.ids)]
            other = [it for it in pend if not (it.ids is None or self._ids_from_camera(it.ids))]
            fb = None
            if self.fallbacks is not None and own:
                fb = self.fallbacks.rows_for((W, H), len(own), self.device)
            if own:
                cams = self._upload_cams([it.cam for it in own], cur)
                ready = [it.ready for it in own if it.ready is not None]
                self._fold([it.probs for it in own], cams, W, H, fb, cur, ready=ready)
                if fb is not None:
                    for k, it in enumerate(own):
                        self.fallbacks[it.fallback_key] = (fb, k)
            for it in other:
                self._fold_rows(it, W, H, cur)

    def _upload_cams(self, rows, cur):
        """(B, 16) device cameras through a reusable pinned host ring: a copy from
        pageable memory would wait for the stream, stalling the host behind the
        batches already queued instead of overlapping them."""
        ring = self._cam_ring
        if ring is None or ring[0].shape[1] < len(rows):
            n = max(len(rows), MAX_BATCH_CAP)
            ring = self._cam_ring = (torch.empty((2, n, 16), dtype=torch.float64).pin_memory(), [None, None], [0])
        host, done, nxt = ring
        slot = nxt[0]
        nxt[0] ^= 1
        if done[slot] is not None:
            done[slot].synchronize()  # the copy that last read this slot has finished
        buf = host[slot, : len(rows)]
        buf.numpy()[:] = np.stack(rows)
        with torch.cuda.stream(cur):
            cams = buf.to(self.device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cur)
        done[slot] = ev
        return cams

    def _ids_from_camera(self, ids):
        src = getattr(ids, "_source", None)
        return src is not None and (src[0] is self.scene or src[0].matches(self.mesh, self.layout))

    def _fold_rows(self, it, W, H, cur):
        """One frame with an explicit IdImage (its rows on this layout)."""
        tex = self._tex
        tex._push_host()
        hw = H * W
        rows = it.ids.rows_on(self.scene).view(1, hw)
        if it.ready is not None:
            cur.wait_event(it.ready)
        hits = None
        if self.weight_mode != "pixels_iid":
            hits = self.scene.hits(1)
            N.call("tfb_count_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle(cur))
        fb = torch.empty(hw, dtype=torch.int32, device=self.device) if self.fallbacks is not None else None
        parr, _keep = N.ptr_array([it.probs.data_ptr()])
        N.call("tfb_fuse", N.ptr(rows), hw, 1, parr, self.num_classes, N.ptr(hits), None, tex.total_texels,
               N.AGG_IDS[tex.aggregator], N.WMODE_IDS[self.weight_mode], float(self.alpha or 0.0),
               N.ptr(tex._accum), tex.accum_kind, tex.stride, N.ptr(tex._counts), N.ptr(fb), N.stream_handle(cur))
        if hits is not None:
            N.call("tfb_clear_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle(cur))
        if fb is not None:
            self.fallbacks[it.fallback_key] = (fb.view(1, hw), 0)
        tex._h_accum = tex._h_counts = None
        self.frames_added += 1

    # -- exchange ------------------------------------------------------------------------
    def allreduce(self, group=None):
        """Sum accumulators and counts over all ranks (one NCCL all-reduce each)."""
        from .dist import allreduce_sum_

        tex = self.texture
        tex._push_host()
        allreduce_sum_([tex._accum, tex._counts], group)
        tex._h_accum = tex._h_counts = None

    def finalize_distributed(self, group=None):
        """Multi-rank end of a job: sum reduce-scatter of the accumulator rows,
        each rank finalizes its slice on its GPU, int32 labels all-gathered
        (dist.reduce_scatter_finalize).  Afterwards labels() / render() work on
        every rank; the per-texel distributions (get()) are not gathered."""
        from .dist import reduce_scatter_finalize

        tex = self.texture
        if tex.finalized:
            raise RuntimeError("texture is already finalized")
        tex._push_host()
        c = tex.num_classes

        def finalize_slice(acc, cnt):
            n = int(acc.shape[0])
            labels = torch.empty(n, dtype=torch.int32, device=acc.device)
            unobs = torch.empty(n, dtype=torch.uint8, device=acc.device)
            N.call("tfb_finalize", N.ptr(acc), tex.accum_kind, tex.stride, N.ptr(cnt), n, c,
                   N.AGG_IDS[tex.aggregator], None, N.ptr(unobs), N.ptr(labels),
                   N.stream_handle(torch.cuda.current_stream(acc.device)))
            return labels

        with torch.cuda.device(self.device):
            tex._labels = reduce_scatter_finalize(tex._accum, tex._counts, finalize_slice, group)
        tex._rows = None
        tex._unobs = None
        tex.finalized = True
        return tex._labels

    # -- results -------------------------------------------------------------------------
    def _finalize(self):
        from .fusion import finalize

        tex = self.texture
        if not tex.finalized:
            with torch.cuda.device(self.device):
                finalize(tex)

    def get(self, host=False):
        """Finalize once; per-texel class distributions (n_x, c) float32."""
        self._finalize()
        return self._tex.rows if host else self._tex.rows_device

    def labels(self, host=False):
        self._finalize()
        return N.host_copy(self._tex.labels_device) if host else self._tex.labels_device

    def render(self, cameras, width=None, height=None, fallback=None, host=False, stream=None):
        """Label images (B, H, W) int32 for the given cameras (renderback.py:28-56)."""
        self._finalize()
        W, H = _sizes(cameras, width, height)
        with torch.cuda.device(self.device):
            cur = stream if stream is not None else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(cur):
                cams = _cams_array(cameras).to(self.device, non_blocking=True)
                B = int(cams.shape[0])
                hw = H * W
                out = torch.empty((B, hw), dtype=torch.int32, device=self.device)
                fb_all = None
                if fallback is not None:
                    fb_all = torch.as_tensor(fallback).to(self.device, torch.int32).reshape(B, hw)
            labels = self._tex.labels_device
            mb = self._batch_for(W, H)
            for b0 in range(0, B, mb):
                b = min(mb, B - b0)
                rows = self.scene.buffer("render_rows", (mb, hw), torch.int32)[:b]
                self.scene.rasterize(cams[b0:b0 + b], W, H, rows, stream=cur)
                fb = fb_all[b0:b0 + b].contiguous() if fb_all is not None else None
                render_labels_device(labels, rows, hw, b, fb, out[b0:b0 + b], cur)
        out = out.view(B, H, W)
        return N.host_copy(out) if host else out

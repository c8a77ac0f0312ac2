"""MeshAnnotation-style fusion: ``add(probs, camera)`` / ``get()`` / ``render(camera)``.

The batched, device-resident front end of the hot path (BASELINE north star):
for each batch of up to ``max_batch`` frames of one size it issues the
stream-ordered launches of tfb_rasterize (vertex outcodes, cull, setup +
tile binning, tile raster with the per-frame texel hit counts fused into its
epilogue), one tfb_fuse scatter-add and the hit-counter reset, and never
synchronizes with the host.  Host inputs are copied on a separate stream
into double-buffered device staging, overlapping the previous batch's
kernels.  ``get()`` finalizes once (tfb_finalize) and returns the per-texel
rows; ``render`` rasterizes the requested cameras and gathers labels
(tfb_render).  Multi-GPU: each rank adds its own frames, then
``finalize_distributed()`` (reduce-scatter, slice finalize, label
all-gather) or ``allreduce()`` (then ``get()``).

It is a thin layer over the same ProbabilityTexture the reference-compatible
functions use (fusion.py / session.py), so textures and results interchange.
"""

import numpy as np
import torch

from . import _native as N
from .device import scene_for
from .fusion import init_texture, parse_weight_mode
from .geometry import pack_camera, uniform_layout
from .renderback import render_labels_device


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


class MeshAnnotation:
    """Fuse per-frame class probabilities onto a mesh's texels on the GPU."""

    def __init__(self, mesh, layout=None, num_classes=None, aggregator="mul", weight_mode="images_iid",
                 accum_dtype="float32", max_batch=8, device=None, memory_budget=None, overlap=False,
                 fuse_ctas_per_sm=None):
        if num_classes is None:
            raise ValueError("num_classes is required")
        self.mesh = mesh
        self.layout = layout if layout is not None else uniform_layout(mesh, 1)
        self.num_classes = int(num_classes)
        self.weight_mode, self.alpha = parse_weight_mode(weight_mode)
        budget = memory_budget if memory_budget is not None else float("inf")
        self.texture = init_texture(self.layout, self.num_classes, aggregator, budget, accum_dtype, device)
        self.scene = scene_for(mesh, self.layout, self.texture.device)
        self.device = self.scene.device
        self.max_batch = int(max_batch)
        self._staging = [None, None]  # device staging for host inputs (double-buffered)
        self._stage_free = [None, None]
        self._stage_slot = 0
        self._copy_stream = None
        self.frames_added = 0
        # Overlap mode: batch k+1 is rasterized on a side stream while batch k
        # is scatter-added on the caller's stream (double-buffered row / hit
        # images); the scatter kernel is capped at fuse_ctas_per_sm resident
        # CTAs so rasterizer CTAs can share the SMs.
        self.overlap = bool(overlap)
        self._side = torch.cuda.Stream(self.device) if self.overlap else None
        self._free = [None, None]
        if fuse_ctas_per_sm is None:
            fuse_ctas_per_sm = 2 if self.overlap else 0
        N.call("tfb_set_option", 1, int(fuse_ctas_per_sm))
        # optional list receiving (frames, ev_raster_start, ev_raster_end, ev_fuse_start, ev_fuse_end)
        self.profile = None

    @staticmethod
    def _event(stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def reset(self):
        """Zero the accumulator and counts for a new fusion job (same layout)."""
        tex = self.texture
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
                 accum=tex._accum[:, : self.num_classes].cpu().numpy(), counts=tex._counts.cpu().numpy(),
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
        from .errors import DataError

        tex = self.texture
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
            tex._accum[:, : self.num_classes].copy_(torch.as_tensor(accum).to(self.device, tex.dtype))
            tex._counts.copy_(torch.as_tensor(counts).to(self.device, tex._counts.dtype))
            self.frames_added = int(z["frames_added"])

    # -- accumulation ------------------------------------------------------------------
    def _probs_batch(self, probs, b, H, W):
        """Per-frame device pointers for b frames.  Contiguous float32 device
        tensors are used in place; anything else (host arrays, pinned host
        tensors) is copied into one of two device staging buffers on a copy
        stream, so the copy of batch k+1 overlaps the kernels of batch k.
        Returns (pointers, keep-alive list, copy-done event or None, staging slot)."""
        c = self.num_classes
        if isinstance(probs, (list, tuple)):
            items = list(probs)
        else:
            items = [probs[i] for i in range(b)] if probs.ndim == 4 else [probs]
        for p in items:
            if tuple(p.shape) != (H, W, c):
                from .errors import DataError

                raise DataError("probability array shape %s does not match expected %s"
                                % (tuple(p.shape), (H, W, c)))
        need_stage = [i for i, p in enumerate(items) if not (isinstance(p, torch.Tensor) and p.is_cuda
                                                             and p.dtype == torch.float32 and p.is_contiguous()
                                                             and p.data_ptr() % 16 == 0)]
        ready, slot = None, None
        if need_stage:
            shape = (self.max_batch, H, W, c)
            slot = self._stage_slot
            self._stage_slot ^= 1
            if self._staging[slot] is None or tuple(self._staging[slot].shape) != shape:
                self._staging[slot] = torch.empty(shape, dtype=torch.float32, device=self.device)
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream(self.device)
            cs = self._copy_stream
            if self._stage_free[slot] is not None:
                cs.wait_event(self._stage_free[slot])  # the scatter that last read this buffer is done
            with torch.cuda.stream(cs):
                for i in need_stage:
                    p, dst = items[i], self._staging[slot][i]
                    if isinstance(p, torch.Tensor):
                        dst.copy_(p, non_blocking=True)
                    else:
                        dst.copy_(torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32)), non_blocking=True)
                    items[i] = dst
            ready = torch.cuda.Event()
            ready.record(cs)
        return [p.data_ptr() for p in items], items, ready, slot

    def add_batch(self, probs, cameras, width=None, height=None, fallback_out=None, stream=None):
        """Fold B frames: probs (B, H, W, c) tensor/array or a list of (H, W, c);
        cameras a list of CameraFrame or a (B, 16) camera array/tensor.
        fallback_out (optional (B, H*W) int32 device tensor) receives each
        frame's network argmax."""
        tex = self.texture
        if tex.finalized:
            raise RuntimeError("texture is already finalized")
        W, H = _sizes(cameras, width, height)
        cur = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(cur):
            cams_all = _cams_array(cameras).to(self.device, non_blocking=True)
        B = int(cams_all.shape[0])
        hw = H * W
        tex._push_host()
        needs_hits = self.weight_mode != "pixels_iid"
        nslots = 2 if self.overlap else 1
        mb = self.max_batch
        rows_all = self.scene.buffer("rows", (nslots, mb, hw), torch.int32)
        hits_all = (self.scene.buffer("hits2", (nslots, mb, max(tex.total_texels, 1)), torch.int32, zero=True)
                    if needs_hits else None)
        side = self._side if self.overlap else cur
        if self.overlap:
            side.wait_stream(cur)  # cameras and anything queued before this call
            cams_all.record_stream(side)
        for i, b0 in enumerate(range(0, B, mb)):
            b = min(mb, B - b0)
            slot = i % nslots
            chunk = probs[b0:b0 + b]
            ptrs, keep, copied, sslot = self._probs_batch(chunk, b, H, W)
            rows = rows_all[slot, :b]
            hits = hits_all[slot, :b] if needs_hits else None
            if self.overlap and self._free[slot] is not None:
                side.wait_event(self._free[slot])  # the scatter that last read this slot is done
            prof = self.profile
            r0 = self._event(side) if prof is not None else None
            self.scene.rasterize(cams_all[b0:b0 + b], W, H, rows, hits=hits, stream=side)
            r1 = self._event(side) if prof is not None else None
            if self.overlap:
                ready = torch.cuda.Event()
                ready.record(side)
                cur.wait_event(ready)
            if copied is not None:
                cur.wait_event(copied)
            f0 = self._event(cur) if prof is not None else None
            parr, _k = N.ptr_array(ptrs)
            fb = fallback_out[b0:b0 + b] if fallback_out is not None else None
            N.call("tfb_fuse", N.ptr(rows), hw, b, parr, self.num_classes, N.ptr(hits), None, tex.total_texels,
                   N.AGG_IDS[tex.aggregator], N.WMODE_IDS[self.weight_mode], float(self.alpha or 0.0),
                   N.ptr(tex._accum), int(tex.is_f64), tex.stride, N.ptr(tex._counts), N.ptr(fb),
                   N.stream_handle(cur))
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

    def add(self, probs, camera, **kw):
        """Fold one (H, W, c) probability map seen from ``camera``."""
        self.add_batch([probs], [camera] if not isinstance(camera, (list, tuple)) else camera, **kw)

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
            N.call("tfb_finalize", N.ptr(acc), int(tex.is_f64), tex.stride, N.ptr(cnt), n, c,
                   N.AGG_IDS[tex.aggregator], None, N.ptr(unobs), N.ptr(labels), N.stream_handle())
            return labels

        tex._labels = reduce_scatter_finalize(tex._accum, tex._counts, finalize_slice, group)
        tex._rows = None
        tex._unobs = None
        tex.finalized = True
        return tex._labels

    # -- results -------------------------------------------------------------------------
    def _finalize(self):
        from .fusion import finalize

        if not self.texture.finalized:
            finalize(self.texture)

    def get(self, host=False):
        """Finalize once; per-texel class distributions (n_x, c) float32."""
        self._finalize()
        return self.texture.rows if host else self.texture.rows_device

    def labels(self, host=False):
        self._finalize()
        return self.texture.labels_device.cpu().numpy() if host else self.texture.labels_device

    def render(self, cameras, width=None, height=None, fallback=None, host=False, stream=None):
        """Label images (B, H, W) int32 for the given cameras (renderback.py:28-56)."""
        self._finalize()
        W, H = _sizes(cameras, width, height)
        cams = _cams_array(cameras).to(self.device, non_blocking=True)
        B = int(cams.shape[0])
        hw = H * W
        out = torch.empty((B, hw), dtype=torch.int32, device=self.device)
        labels = self.texture.labels_device
        for b0 in range(0, B, self.max_batch):
            b = min(self.max_batch, B - b0)
            rows = self.scene.buffer("render_rows", (self.max_batch, hw), torch.int32)[:b]
            self.scene.rasterize(cams[b0:b0 + b], W, H, rows, stream=stream)
            fb = None
            if fallback is not None:
                fb = torch.as_tensor(fallback).to(self.device, torch.int32).reshape(B, hw)[b0:b0 + b].contiguous()
            render_labels_device(labels, rows, hw, b, fb, out[b0:b0 + b], stream)
        out = out.view(B, H, W)
        return out.cpu().numpy() if host else out

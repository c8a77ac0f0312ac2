"""Per-texel probability accumulation on the GPU (texelfuse/fusion.py).

Same names, arguments, aggregation rules and error behaviour as the
reference: ``init_texture`` / ``compute_pixel_weights`` /
``accumulate_frame`` / ``finalize`` / ``texel_argmax``.  The accumulator,
counts and finalized rows live in device memory; ``tex.accum``,
``tex.counts``, ``tex.rows`` and ``tex.unobserved`` are NumPy views
materialized on access (writes to ``accum``/``counts`` are uploaded before
the next device operation, so the reference's own tests that poke the
texture keep working).

Accumulator precision: ``accum_dtype="float64"`` (default here, matching the
reference's float64 fold and its 1e-6 row tests), ``"float32"`` (the
throughput mode; red.global.add.v4.f32, within 1e-5 relative) or
``"fixed64"`` (int64 fixed point in units of 2^-32: every piece of equal-row
pixels is summed in float64 in a fixed order and added with an integer
atomic, so reruns are bit-identical whatever the scheduling -- the CLI's
``deterministic=true`` and the session API use it).
"""

import numpy as np
import torch

from . import _native as N
from .device import layout_scene
from .errors import CapacityError, DataError

AGGREGATORS = ("sum", "maxsum", "mul")  # fusion.py:34
WEIGHT_MODES = ("pixels_iid", "images_iid", "blend")  # fusion.py:35
MUL_CLAMP = 1e-7  # fusion.py:39
UNKNOWN = -1  # fusion.py:42
DEFAULT_MEMORY_BUDGET = 4 * 1024 ** 3  # fusion.py:44
DEFAULT_ACCUM_DTYPE = "float64"

_DTYPES = {"float32": torch.float32, "float64": torch.float64, torch.float32: torch.float32,
           torch.float64: torch.float64, np.float32: torch.float32, np.float64: torch.float64,
           "fixed64": torch.int64, torch.int64: torch.int64}
FIXED_SCALE = 2.0 ** 32  # TFB_ACCUM_FIXED: accumulator element = round(value * 2^32)
ACCUM_KIND = {torch.float32: 0, torch.float64: 1, torch.int64: 2}  # TFB_ACCUM_F32 / F64 / FIXED


def texture_nbytes(total_texels, num_classes):
    """Reference budget formula: f64 accumulator + f32 rows + i64 counts (fusion.py:65-67)."""
    return total_texels * num_classes * 12 + total_texels * 8


def accum_stride(num_classes, dtype):
    return (num_classes + 3) // 4 * 4 if dtype == torch.float32 else num_classes


class ProbabilityTexture:
    """Device-resident accumulation state for one layout (fusion.py:47-62)."""

    def __init__(self, layout, num_classes, aggregator, accum_dtype=DEFAULT_ACCUM_DTYPE, device=None):
        self.layout = layout
        self.num_classes = int(num_classes)
        self.aggregator = aggregator
        self.finalized = False
        self._scene = layout_scene(layout, device)
        self.device = self._scene.device
        if accum_dtype not in _DTYPES:
            raise ValueError("accum_dtype must be float32, float64 or fixed64, got %r" % (accum_dtype,))
        self.dtype = _DTYPES[accum_dtype]
        self.stride = accum_stride(self.num_classes, self.dtype)
        n = max(int(layout.total_texels), 0)
        self._accum = torch.zeros((max(n, 1), self.stride), dtype=self.dtype, device=self.device)[:n]
        self._counts = torch.zeros(max(n, 1), dtype=torch.int32, device=self.device)[:n]
        self._rows = None
        self._unobs = None
        self._labels = None
        self._h_accum = None
        self._h_counts = None
        self._h_rows = None
        self._h_unobs = None
        self._flush_hook = None  # weak method of a MeshAnnotation / session holding queued frames

    def _flush_pending(self):
        hook = self._flush_hook
        if hook is not None:
            fn = hook()
            if fn is not None:
                fn()

    @property
    def total_texels(self):
        return self.layout.total_texels

    @property
    def is_f64(self):
        return self.dtype == torch.float64

    @property
    def accum_kind(self):
        """C ABI accumulator kind: TFB_ACCUM_F32 (0), TFB_ACCUM_F64 (1), TFB_ACCUM_FIXED (2)."""
        return ACCUM_KIND[self.dtype]

    def accum_values(self, t=None):
        """Accumulator elements (device) as float64 values."""
        t = self._accum[:, : self.num_classes] if t is None else t
        if self.dtype == torch.int64:
            return t.to(torch.float64) / FIXED_SCALE
        return t.to(torch.float64)

    def accum_from_values(self, a):
        """(n_x, c) float64 values → accumulator elements of this texture's kind (device)."""
        t = torch.as_tensor(np.asarray(a, dtype=np.float64)).to(self.device)
        if self.dtype == torch.int64:
            return torch.round(t * FIXED_SCALE).to(torch.int64)
        return t.to(self.dtype)

    # -- host views (reference fields) ---------------------------------------------
    @property
    def accum(self):
        self._flush_pending()
        if self._h_accum is None:
            self._h_accum = self.accum_values().cpu().numpy()
        return self._h_accum

    @accum.setter
    def accum(self, value):
        self._h_accum = np.array(value, dtype=np.float64, copy=True)

    @property
    def counts(self):
        self._flush_pending()
        if self._h_counts is None:
            self._h_counts = self._counts.to(torch.int64).cpu().numpy()
        return self._h_counts

    @counts.setter
    def counts(self, value):
        self._h_counts = np.array(value, dtype=np.int64, copy=True)

    @property
    def rows(self):
        if self._rows is None:
            return None
        if self._h_rows is None:
            self._h_rows = self._rows.cpu().numpy()
        return self._h_rows

    @property
    def unobserved(self):
        if self._unobs is None:
            return None
        if self._h_unobs is None:
            self._h_unobs = self._unobs.cpu().numpy().astype(bool)
        return self._h_unobs

    # -- device views ------------------------------------------------------------------
    @property
    def rows_device(self):
        """(n_x, c) float32 device tensor after finalize."""
        return self._rows

    @property
    def labels_device(self):
        return self._labels

    def accum_device(self):
        self._flush_pending()
        self._push_host()
        return self._accum

    def counts_device(self):
        self._flush_pending()
        self._push_host()
        return self._counts

    def _push_host(self):
        """Fold queued frames, then upload host mirrors (which callers may have
        written) before device work."""
        self._flush_pending()
        if self._h_accum is not None:
            a = np.asarray(self._h_accum, dtype=np.float64)
            if a.shape != (self.total_texels, self.num_classes):
                raise DataError("accumulator shape %s does not match texture" % (a.shape,))
            self._accum[:, : self.num_classes].copy_(self.accum_from_values(a))
            self._h_accum = None
        if self._h_counts is not None:
            self._counts.copy_(torch.as_tensor(np.asarray(self._h_counts, dtype=np.int64)).to(self.device,
                                                                                                 torch.int32))
            self._h_counts = None


def init_texture(layout, num_classes, aggregator="mul", memory_budget=DEFAULT_MEMORY_BUDGET,
                 accum_dtype=DEFAULT_ACCUM_DTYPE, device=None):
    """Zeroed device texture (fusion.py:70-93); same validation and CapacityError text."""
    if aggregator not in AGGREGATORS:
        raise ValueError("unknown aggregator %r (expected one of %s)" % (aggregator, AGGREGATORS))
    if num_classes < 2:
        raise ValueError("num_classes must be >= 2")
    need = texture_nbytes(layout.total_texels, num_classes)
    if need > memory_budget:
        raise CapacityError(
            "probability texture needs %d bytes (%d texels x %d classes) but the memory budget is %d bytes"
            % (need, layout.total_texels, num_classes, memory_budget))
    return ProbabilityTexture(layout, num_classes, aggregator, accum_dtype, device)


def parse_weight_mode(spec):
    """'pixels_iid' | 'images_iid' | 'blend:<a>' | 'blend(<a>)' → (mode, alpha) (fusion.py:96-111)."""
    spec = spec.strip()
    if spec in ("pixels_iid", "images_iid"):
        return spec, None
    for head, tail in (("blend:", ""), ("blend(", ")")):
        if spec.startswith(head) and spec.endswith(tail):
            body = spec[len(head): len(spec) - len(tail)]
            try:
                alpha = float(body)
            except ValueError:
                break
            if not 0.0 <= alpha <= 1.0:
                raise ValueError("blend alpha %g outside [0, 1]" % alpha)
            return "blend", alpha
    raise ValueError("unknown weight mode %r" % spec)


def _check_mode(mode, alpha):
    if mode not in WEIGHT_MODES:
        raise ValueError("unknown weight mode %r (expected one of %s)" % (mode, WEIGHT_MODES))
    if mode == "blend" and (alpha is None or not 0.0 <= alpha <= 1.0):
        raise ValueError("blend weight mode needs alpha in [0, 1]")


class PixelWeights(np.ndarray):
    """compute_pixel_weights result: an (H, W) float64 ndarray (fusion.py:114-142)
    computed on the device, read-only, that remembers how it was derived so
    accumulate_frame can rebuild the same weights on the device from the frame's
    hit counts instead of uploading them.  Arrays derived from it (views,
    arithmetic, copies) are plain writable weights and take the explicit path."""

    def __array_finalize__(self, obj):
        self._spec = None


def _virtual_rows(ids, device):
    """Rows keyed on (triangle, texel) pairs, for weights of IdImages with no layout."""
    if ids._rows is not None:
        return ids._rows, ids._rows_scene.total_texels
    tri = np.asarray(ids.triangle, dtype=np.int64).reshape(-1)
    tex = np.asarray(ids.texel, dtype=np.int64).reshape(-1)
    cov = tri != -1
    rows = np.full(tri.shape, -1, dtype=np.int32)
    if cov.any():
        _, inv = np.unique(tri[cov] << 32 | tex[cov], return_inverse=True)
        rows[cov] = inv.astype(np.int32)
    n = int(rows.max()) + 1 if cov.any() else 1
    return torch.as_tensor(rows).to(device), n


def _weights_on_device(ids, mode, alpha):
    import torch as _t

    ids._ensure_device()
    dev = ids._rows.device if ids._rows is not None else _t.device("cuda", _t.cuda.current_device())
    rows, n = _virtual_rows(ids, dev)
    hw = ids.width * ids.height
    hits = None
    if mode != "pixels_iid":
        hits = _t.zeros(max(n, 1), dtype=_t.int32, device=dev)
        N.call("tfb_count_hits", N.ptr(rows), hw, 1, n, N.ptr(hits), N.stream_handle())
    out = _t.empty(hw, dtype=_t.float64, device=dev)
    N.call("tfb_pixel_weights", N.ptr(rows), hw, 1, N.ptr(hits), n, N.WMODE_IDS[mode], float(alpha or 0.0),
           N.ptr(out), N.stream_handle())
    return out


def compute_pixel_weights(ids, mode, alpha=None):
    """Per-pixel fusion weight for one frame (fusion.py:114-142)."""
    _check_mode(mode, alpha)
    N.require_cuda()
    host = N.host_copy(_weights_on_device(ids, mode, alpha)).reshape(ids.height, ids.width)
    w = host.view(PixelWeights)
    w._spec = (ids, mode, alpha)
    w.flags.writeable = False
    return w


def _probs_device(probs, H, W, c, device):
    """(H*W, c) float32 contiguous 16-byte-aligned device tensor."""
    if isinstance(probs, torch.Tensor):
        t = probs.detach()
        if tuple(t.shape) != (H, W, c):
            raise DataError("probability image shape %s does not match frame %dx%d with %d classes"
                            % (tuple(t.shape), W, H, c))
        t = t.to(device=device, dtype=torch.float32).contiguous()
    else:
        a = np.asarray(probs)
        if a.shape != (H, W, c):
            raise DataError("probability image shape %s does not match frame %dx%d with %d classes"
                            % (a.shape, W, H, c))
        t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(device)
    if t.data_ptr() % 16:
        t = t.clone()
    return t.view(H * W, c)


def _on_texture_device(fn):
    """Run a texture operation with the texture's GPU current, so the C ABI
    launches there and N.stream_handle() names that device's stream."""
    import functools

    @functools.wraps(fn)
    def run(tex, *args, **kw):
        dev = getattr(tex, "device", None)
        if isinstance(dev, torch.device) and dev.type == "cuda":
            with torch.cuda.device(dev):
                return fn(tex, *args, **kw)
        return fn(tex, *args, **kw)

    return run


@_on_texture_device
def accumulate_frame(tex, ids, probs, weights):
    """Fold one frame's class distributions into the texture (fusion.py:145-183)."""
    if tex.finalized:
        raise RuntimeError("texture is already finalized")
    H, W = ids.height, ids.width
    c = tex.num_classes
    pshape = tuple(probs.shape)
    if pshape != (H, W, c):
        raise DataError("probability image shape %s does not match frame %dx%d with %d classes"
                        % (pshape, W, H, c))
    wshape = tuple(weights.shape)
    if wshape != (H, W):
        raise DataError("weight image shape %s does not match frame" % (wshape,))
    tex._push_host()
    scene = tex._scene
    rows = ids.rows_on(scene)
    p = _probs_device(probs, H, W, c, tex.device)
    hw = H * W
    hits = None
    wdev = None
    spec = getattr(weights, "_spec", None) if isinstance(weights, PixelWeights) else None
    if spec is not None and spec[0] is ids and not weights.flags.writeable:
        mode, alpha = spec[1], spec[2]
        if mode != "pixels_iid":
            hits = scene.hits(1)
            N.call("tfb_count_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle())
    else:
        mode, alpha = "explicit", 0.0
        w = weights
        if isinstance(w, torch.Tensor):
            wdev = w.detach().to(device=tex.device, dtype=torch.float64).contiguous().view(-1)
        else:
            wdev = torch.as_tensor(np.ascontiguousarray(w, dtype=np.float64)).to(tex.device).view(-1)
    ptrs, _keep = N.ptr_array([p.data_ptr()])
    N.call("tfb_fuse", N.ptr(rows), hw, 1, ptrs, c, N.ptr(hits), N.ptr(wdev), tex.total_texels,
           N.AGG_IDS[tex.aggregator], N.WMODE_IDS[mode], float(alpha or 0.0), N.ptr(tex._accum), tex.accum_kind,
           tex.stride, N.ptr(tex._counts), None, N.stream_handle())
    if hits is not None:
        N.call("tfb_clear_hits", N.ptr(rows), hw, 1, tex.total_texels, N.ptr(hits), N.stream_handle())
    tex._h_accum = None
    tex._h_counts = None
    return tex


@_on_texture_device
def finalize(tex):
    """Normalize accumulated rows into per-texel distributions (fusion.py:186-210)."""
    if tex.finalized:
        raise RuntimeError("texture is already finalized")
    tex._push_host()
    n, c = tex.total_texels, tex.num_classes
    d = tex.device
    tex._rows = torch.empty((n, c), dtype=torch.float32, device=d)
    tex._unobs = torch.empty(n, dtype=torch.uint8, device=d)
    tex._labels = torch.empty(n, dtype=torch.int32, device=d)
    N.call("tfb_finalize", N.ptr(tex._accum), tex.accum_kind, tex.stride, N.ptr(tex._counts), n, c,
           N.AGG_IDS[tex.aggregator], N.ptr(tex._rows), N.ptr(tex._unobs), N.ptr(tex._labels), N.stream_handle())
    tex.finalized = True
    tex._h_rows = tex._h_unobs = None
    return tex


def texel_argmax(tex):
    """Most probable class per texel, UNKNOWN where unobserved (fusion.py:213-222)."""
    if not tex.finalized:
        raise RuntimeError("texture must be finalized before argmax")
    return N.host_copy(tex._labels)

"""tfb_fuse kernel coverage beyond the scene tests: both scatter-add kernels
(the specialised float32 / count-weight / c % 4 == 0 kernel and the general
one, selected with TFB_OPT_FUSE_FAST) against the float64 oracle
(oracle.accumulate_frame, fusion.py:145-183) on synthetic row images with
texel runs, partial last chunks, several quad passes (c = 132), class counts
that are not a multiple of 4 (masked quads, bulk-copy tails), and the
probability values the clip / log paths care about: 0, tiny, exactly 1,
above 1, negative, NaN and values just below 1 (log1p series path)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2111_11103_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu

P = ctypes.c_void_p
TFB_OPT_FUSE_FAST = 2


def _rows(rng, nframes, hw, n_x):
    """Row images made of runs (1..9 pixels) on random texels, ~15% uncovered."""
    out = np.empty((nframes, hw), np.int32)
    for f in range(nframes):
        i = 0
        while i < hw:
            n = int(rng.integers(1, 10))
            r = -1 if rng.random() < 0.15 else int(rng.integers(0, n_x))
            out[f, i:i + n] = r
            i += n
    return out


def _probs(rng, nframes, hw, c, special):
    logits = rng.normal(size=(nframes, hw, c)) * 2.0
    p = np.exp(logits - logits.max(axis=2, keepdims=True))
    p = (p / p.sum(axis=2, keepdims=True)).astype(np.float32)
    if special:
        flat = p.reshape(-1)
        m = flat.size
        pick = lambda k: rng.choice(m, size=k, replace=False)  # noqa: E731
        flat[pick(m // 50)] = 0.0
        flat[pick(m // 200)] = 1e-9
        flat[pick(m // 200)] = 1.0
        flat[pick(m // 500)] = 1.5
        flat[pick(m // 500)] = -0.25
        flat[pick(m // 50)] = rng.uniform(0.9, 0.99999, size=m // 50).astype(np.float32)
        flat[pick(3)] = np.nan
    return p


def _run(rows, probs, n_x, agg, wm, alpha, fast):
    lib = N.load()
    nframes, hw = rows.shape
    c = probs.shape[2]
    stride = (c + 3) // 4 * 4
    dev = torch.device("cuda")
    rows_d = torch.as_tensor(rows, device=dev)
    pd = [torch.as_tensor(probs[f], device=dev).contiguous() for f in range(nframes)]
    ptrs = (P * nframes)(*[t.data_ptr() for t in pd])
    hits = torch.zeros((nframes, n_x), dtype=torch.int32, device=dev)
    acc = torch.zeros((n_x, stride), dtype=torch.float32, device=dev)
    cnt = torch.zeros(n_x, dtype=torch.int32, device=dev)
    fb = torch.full((nframes, hw), -7, dtype=torch.int32, device=dev)
    stream = P(torch.cuda.current_stream().cuda_stream)
    N.check(lib.tfb_set_option(TFB_OPT_FUSE_FAST, 1 if fast else 0))
    try:
        N.check(lib.tfb_count_hits(P(rows_d.data_ptr()), hw, nframes, n_x, P(hits.data_ptr()), stream))
        N.check(lib.tfb_fuse(P(rows_d.data_ptr()), hw, nframes, ctypes.cast(ptrs, P), c, P(hits.data_ptr()), None,
                             n_x, N.AGG_IDS[agg], N.WMODE_IDS[wm], alpha, P(acc.data_ptr()), 0, stride,
                             P(cnt.data_ptr()), P(fb.data_ptr()), stream))
        torch.cuda.synchronize()
    finally:
        lib.tfb_set_option(TFB_OPT_FUSE_FAST, 1)
    return acc.cpu().numpy()[:, :c], cnt.cpu().numpy(), fb.cpu().numpy()


def _oracle(rows, probs, n_x, agg, wm, alpha):
    acc = np.zeros((n_x, probs.shape[2]))
    cnt = np.zeros(n_x, np.int64)
    offsets = np.arange(n_x, dtype=np.int64)
    for f in range(rows.shape[0]):
        tri = rows[f]
        texel = np.zeros_like(tri)
        w = O.compute_pixel_weights(tri, texel, wm, alpha if wm == "blend" else None)
        O.accumulate_frame(acc, cnt, offsets, tri, texel, probs[f], w, agg)
    return acc, cnt


def _check(got, ref, scale, tol=1e-5):
    """float32 accumulation bound: relative to the sum of |terms| (scale), floored at 1e-3."""
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    err = np.abs(got[ok] - ref[ok]) / np.maximum(np.maximum(np.abs(scale[ok]), np.abs(ref[ok])), 1e-3)
    assert err.max(initial=0.0) < tol, err.max()


def _scale(rows, probs, n_x, agg, wm, alpha):
    if agg == "mul":  # all terms are <= 0: no cancellation
        return np.abs(_oracle(rows, probs, n_x, agg, wm, alpha)[0])
    return _oracle(rows, np.abs(probs), n_x, agg, wm, alpha)[0]


@pytest.mark.parametrize("fast", [True, False])
@pytest.mark.parametrize("c", [3, 4, 7, 13, 19, 20, 23, 40, 41, 99, 132, 300, 601])
@pytest.mark.parametrize("agg", ["sum", "maxsum", "mul"])
def test_fuse_kernels_vs_oracle(fast, c, agg):
    rng = np.random.default_rng(1000 + c)
    nframes, hw, n_x = 3, 61 * 37, 300
    rows = _rows(rng, nframes, hw, n_x)
    probs = _probs(rng, nframes, hw, c, special=True)
    for wm, alpha in (("images_iid", 0.0), ("pixels_iid", 0.0), ("blend", 0.3)):
        got, cnt, fb = _run(rows, probs, n_x, agg, wm, alpha, fast)
        ref, cref = _oracle(rows, probs, n_x, agg, wm, alpha)
        np.testing.assert_array_equal(cnt, cref)
        _check(got, ref, _scale(rows, probs, n_x, agg, wm, alpha))
    np.testing.assert_array_equal(fb, probs.argmax(axis=2))


def test_fuse_fast_many_frames_and_launch_split():
    """More frames than one launch carries (256): the frame loop and pointer table."""
    rng = np.random.default_rng(5)
    nframes, hw, n_x, c = 261, 32 * 20 + 5, 64, 8
    rows = _rows(rng, nframes, hw, n_x)
    probs = _probs(rng, nframes, hw, c, special=False)
    got, cnt, _ = _run(rows, probs, n_x, "mul", "images_iid", 0.0, True)
    ref, cref = _oracle(rows, probs, n_x, "mul", "images_iid", 0.0)
    np.testing.assert_array_equal(cnt, cref)
    _check(got, ref, ref)


def test_fuse_fast_and_general_agree_on_long_runs():
    """Whole chunks on one texel (product pieces of 5 pixels in the fast kernel, 4 in the general one)."""
    rng = np.random.default_rng(9)
    hw, c = 32 * 64, 40
    rows = np.repeat(np.arange(hw // 256, dtype=np.int32), 256)[None, :]
    probs = _probs(rng, 1, hw, c, special=False)
    a, ca, _ = _run(rows, probs, hw // 256, "mul", "blend", 0.5, True)
    b, cb, _ = _run(rows, probs, hw // 256, "mul", "blend", 0.5, False)
    ref, cref = _oracle(rows, probs, hw // 256, "mul", "blend", 0.5)
    np.testing.assert_array_equal(ca, cref)
    np.testing.assert_array_equal(cb, cref)
    _check(a, ref, ref)
    _check(b, ref, ref)


def test_fuse_fast_products_at_the_clip_floor():
    """Long runs whose values sit at (and just above) the clip floor 1e-7: a
    5-pixel product piece reaches 1e-35, still a normal float32, so no clip
    redo and no underflow; plus values just below the floor (clip redo)."""
    rng = np.random.default_rng(11)
    hw, c = 32 * 40, 8
    rows = np.repeat(np.arange(hw // 160, dtype=np.int32), 160)[None, :]
    probs = np.full((1, hw, c), 1e-7, dtype=np.float32)
    probs[0, :, 0] = 1.0 - 7e-7
    probs[0, ::7, 3] = np.float32(1.0000001e-7)
    probs[0, 5::11, 5] = np.float32(0.99e-7)  # below the floor: np.clip raises it
    for agg in ("mul", "sum"):
        got, cnt, _ = _run(rows, probs, hw // 160, agg, "images_iid", 0.0, True)
        ref, cref = _oracle(rows, probs, hw // 160, agg, "images_iid", 0.0)
        np.testing.assert_array_equal(cnt, cref)
        _check(got, ref, _scale(rows, probs, hw // 160, agg, "images_iid", 0.0))


@pytest.mark.parametrize("fast", [True, False])
@pytest.mark.parametrize("c", [7, 8, 19, 40])
def test_fused_argmax_ties_and_nan(fast, c):
    """The fused network argmax / per-pixel maximum (cli.py:293, fusion.py:174), read as 16-byte
    quads when c % 4 == 0: NumPy's rule must hold -- the first NaN wins, else the FIRST maximum
    (many exact ties here)."""
    rng = np.random.default_rng(77 + c)
    nframes, hw, n_x = 2, 32 * 23 + 9, 50
    rows = _rows(rng, nframes, hw, n_x)
    probs = (np.round(rng.random((nframes, hw, c)) * 4) / 4).astype(np.float32)  # values in {0, .25, ..., 1}
    flat = probs.reshape(-1)
    flat[rng.choice(flat.size, size=flat.size // 97, replace=False)] = np.nan
    for agg in ("sum", "maxsum"):
        got, cnt, fb = _run(rows, probs, n_x, agg, "pixels_iid", 0.0, fast)
        np.testing.assert_array_equal(fb, probs.argmax(axis=2))
        ref, cref = _oracle(rows, probs, n_x, agg, "pixels_iid", 0.0)
        np.testing.assert_array_equal(cnt, cref)
        _check(got, ref, _scale(rows, probs, n_x, agg, "pixels_iid", 0.0))


@pytest.mark.parametrize("c", [8, 40])
def test_fused_argmax_infinities(c):
    """The strict-greater argmax pass with its NaN-detecting running sum: +inf / -inf classes
    (inf is a maximum, -inf never; +inf and -inf in one pixel make the sum NaN and take the
    exact pass), NaN, and all-equal pixels -- NumPy's argmax either way."""
    rng = np.random.default_rng(31 + c)
    nframes, hw, n_x = 1, 32 * 12 + 5, 20
    rows = _rows(rng, nframes, hw, n_x)
    probs = rng.random((nframes, hw, c)).astype(np.float32)
    flat = probs.reshape(-1)
    flat[rng.choice(flat.size, size=flat.size // 30, replace=False)] = np.inf
    flat[rng.choice(flat.size, size=flat.size // 30, replace=False)] = -np.inf
    flat[rng.choice(flat.size, size=flat.size // 200, replace=False)] = np.nan
    probs[0, :7] = 0.5  # all-equal pixels: index 0
    for fast in (True, False):
        _, _, fb = _run(rows, probs, n_x, "sum", "pixels_iid", 0.0, fast)
        np.testing.assert_array_equal(fb, probs.argmax(axis=2))


def _run64(rows, probs, n_x, agg, wm, alpha, weights=None):
    """tfb_fuse into a float64 accumulator (the reference's precision, fusion.py:145-183)."""
    lib = N.load()
    nframes, hw = rows.shape
    c = probs.shape[2]
    dev = torch.device("cuda")
    rows_d = torch.as_tensor(rows, device=dev)
    pd = [torch.as_tensor(probs[f], device=dev).contiguous() for f in range(nframes)]
    ptrs = (P * nframes)(*[t.data_ptr() for t in pd])
    hits = torch.zeros((nframes, n_x), dtype=torch.int32, device=dev)
    acc = torch.zeros((n_x, c), dtype=torch.float64, device=dev)
    cnt = torch.zeros(n_x, dtype=torch.int32, device=dev)
    wd = torch.as_tensor(weights, device=dev) if weights is not None else None
    stream = P(torch.cuda.current_stream().cuda_stream)
    N.check(lib.tfb_count_hits(P(rows_d.data_ptr()), hw, nframes, n_x, P(hits.data_ptr()), stream))
    N.check(lib.tfb_fuse(P(rows_d.data_ptr()), hw, nframes, ctypes.cast(ptrs, P), c, P(hits.data_ptr()),
                         P(wd.data_ptr()) if wd is not None else None, n_x, N.AGG_IDS[agg],
                         N.WMODE_IDS["explicit" if wd is not None else wm], alpha, P(acc.data_ptr()), 1, c,
                         P(cnt.data_ptr()), None, stream))
    torch.cuda.synchronize()
    return acc.cpu().numpy(), cnt.cpu().numpy()


@pytest.mark.parametrize("c", [5, 13, 19, 40, 41, 132])
def test_float64_accumulator_log_within_1e12(c):
    """The float64 accumulator's per-piece log and float-domain clip (fuse.cu clip_mul64)
    against NumPy's log(clip(p, 1e-7, 1)) (fusion.py:177): 1e-12 relative, with values at and
    around 1, at the clip floor, below it, above 1 and NaN; piecewise products (count weights)
    and per-pixel terms (explicit weights)."""
    rng = np.random.default_rng(500 + c)
    nframes, hw, n_x = 2, 32 * 41 + 3, 120
    rows = _rows(rng, nframes, hw, n_x)
    probs = _probs(rng, nframes, hw, c, special=True)
    flat = probs.reshape(-1)
    flat[rng.choice(flat.size, size=flat.size // 40, replace=False)] = np.float32(1e-7)
    flat[rng.choice(flat.size, size=flat.size // 40, replace=False)] = np.float32(0.99999994)
    flat[rng.choice(flat.size, size=flat.size // 40, replace=False)] = np.nextafter(np.float32(1e-7), np.float32(0))
    for wm, alpha in (("images_iid", 0.0), ("blend", 0.25), ("pixels_iid", 0.0)):
        got, cnt = _run64(rows, probs, n_x, "mul", wm, alpha)
        ref, cref = _oracle(rows, probs, n_x, "mul", wm, alpha)
        np.testing.assert_array_equal(cnt, cref)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    w = rng.uniform(0.1, 3.0, size=(nframes, hw))
    got, _ = _run64(rows, probs, n_x, "mul", "explicit", 0.0, weights=w)
    ref = np.zeros((n_x, c))
    cref = np.zeros(n_x, np.int64)
    for f in range(nframes):
        O.accumulate_frame(ref, cref, np.arange(n_x, dtype=np.int64), rows[f], np.zeros_like(rows[f]), probs[f],
                           w[f], "mul")
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("agg", ["sum", "maxsum"])
@pytest.mark.parametrize("c", [7, 19, 40, 41, 132])
def test_float64_accumulator_sum_rules(c, agg):
    """float64 accumulators for sum / maxsum (k_fuse_fast D64 mode for c <= 128, k_fuse above):
    the reference's per-pixel w * p (maxsum: p where it equals the pixel's max, ties kept)
    summed in double, at 1e-12 relative, special values and NaN included."""
    rng = np.random.default_rng(1700 + c)
    nframes, hw, n_x = 2, 32 * 37 + 11, 150
    rows = _rows(rng, nframes, hw, n_x)
    probs = _probs(rng, nframes, hw, c, special=True)
    flat = probs.reshape(-1)
    flat[rng.choice(flat.size, size=flat.size // 20, replace=False)] = 0.25  # max ties
    for wm, alpha in (("images_iid", 0.0), ("blend", 0.3), ("pixels_iid", 0.0)):
        got, cnt = _run64(rows, probs, n_x, agg, wm, alpha)
        ref, cref = _oracle(rows, probs, n_x, agg, wm, alpha)
        np.testing.assert_array_equal(cnt, cref)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("agg", ["mul", "sum", "maxsum"])
@pytest.mark.parametrize("c", [13, 40, 41])
def test_float64_accumulator_long_runs(c, agg):
    """The float64 product rule (k_fuse_fast D64 mode: no 5-pixel cut, a piece runs to the next
    row change or pixel-group start) over runs of 20-70 pixels crossing chunk boundaries, values
    near the clip floor and near 1 (products of up to 32 values in double), and a partial last
    chunk: 1e-12 relative to NumPy's per-pixel log."""
    rng = np.random.default_rng(1300 + c)
    hw, n_x = 32 * 30 + 7, 40
    runs = np.repeat(np.arange(n_x, dtype=np.int32), 25)[:hw]
    rows = np.stack([runs, runs[::-1].copy()])
    rows[:, 100:130] = -1
    probs = _probs(rng, 2, hw, c, special=False)
    probs[0, :, 0] = np.float32(1.5e-7)
    probs[1, ::3, 1] = np.float32(0.999999)
    for wm, alpha in (("images_iid", 0.0), ("blend", 0.4)):
        got, cnt = _run64(rows, probs, n_x, agg, wm, alpha)
        ref, cref = _oracle(rows, probs, n_x, agg, wm, alpha)
        np.testing.assert_array_equal(cnt, cref)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("c", [7, 19, 40, 41])
@pytest.mark.parametrize("agg", ["sum", "maxsum", "mul"])
def test_fuse_piece_per_pixel_chunks(c, agg):
    """Chunks where nearly every pixel is its own piece (tiny triangles: configs[4]), mixed with
    long-run chunks in the same launch, special values included."""
    rng = np.random.default_rng(900 + c)
    nframes, hw, n_x = 2, 32 * 50 + 13, 5000
    rows = rng.integers(0, n_x, size=(nframes, hw)).astype(np.int32)  # a new row at every pixel
    rows[:, ::17] = -1
    rows[:, 32 * 10: 32 * 20] = np.repeat(np.arange(40, dtype=np.int32), 8)[None, :]  # long runs too
    probs = _probs(rng, nframes, hw, c, special=True)
    for wm, alpha in (("images_iid", 0.0), ("blend", 0.3)):
        got, cnt, fb = _run(rows, probs, n_x, agg, wm, alpha, True)
        ref, cref = _oracle(rows, probs, n_x, agg, wm, alpha)
        np.testing.assert_array_equal(cnt, cref)
        _check(got, ref, _scale(rows, probs, n_x, agg, wm, alpha))
    np.testing.assert_array_equal(fb, probs.argmax(axis=2))


def test_log_f64_against_numpy():
    """The table-driven float64 log of the float64-accumulator scatter-add
    (csrc/log_f64.cuh) against NumPy's log: within 2 ulp over random arguments
    across the whole product range, around 1 (no cancellation), at powers of two
    and at every reduction-interval boundary; special arguments (0, negative,
    subnormal, inf, NaN) follow libdevice / NumPy."""
    rng = np.random.default_rng(7)
    xs = [np.exp(rng.uniform(np.log(1e-300), 0.0, 200000)),            # products of clipped probabilities
          1.0 - np.exp(rng.uniform(np.log(1e-16), np.log(0.3), 20000)),  # just below 1
          1.0 + np.exp(rng.uniform(np.log(1e-16), np.log(0.3), 20000)),  # just above 1
          np.ldexp(1.0, np.arange(-1022, 1023)).astype(np.float64),
          rng.uniform(1e-7, 1.0, 20000)]
    # interval boundaries of z = x * 2^-k in [0.6875, 1.375) and their neighbours
    edges = 0.6875 * (1.0 + np.arange(129) / 128.0)
    edges = np.concatenate([edges[edges < 1.0], 1.0 + (np.arange(49) / 128.0)])
    edges = np.concatenate([edges, np.nextafter(edges, 0.0), np.nextafter(edges, 2.0)])
    for s in (-3, -1, 0, 1, 3):
        xs.append(edges * 2.0 ** s)
    x = np.concatenate(xs).astype(np.float64)
    x = x[(x > 0) & np.isfinite(x)]
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    N.call("tfb_test_log_f64", N.ptr(xd), N.ptr(yd), x.size, N.stream_handle())
    y = yd.cpu().numpy()
    ref = np.log(x)
    ulp = np.spacing(np.abs(ref))
    err = np.abs(y - ref) / ulp
    assert err.max() <= 2.0, (err.max(), x[np.argmax(err)])
    assert np.all(y[x == 1.0] == 0.0)
    special = np.array([0.0, -0.0, -1.0, 5e-324, 1e-310, np.inf, np.nan, 2.0 ** -1022], dtype=np.float64)
    sd = torch.as_tensor(special, device="cuda")
    so = torch.empty_like(sd)
    N.call("tfb_test_log_f64", N.ptr(sd), N.ptr(so), special.size, N.stream_handle())
    got = so.cpu().numpy()
    with np.errstate(divide="ignore", invalid="ignore"):
        want = np.log(special)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    np.testing.assert_allclose(got[ok], want[ok], rtol=1e-15)

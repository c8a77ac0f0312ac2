"""tfb_finalize (fusion.py:186-222) against the NumPy oracle for class counts on
both sides of the 8-lanes-per-texel / warp-per-texel split (c <= 64 / > 64),
float32 and float64 accumulators, all aggregators, unobserved texels, NaN
and tied rows."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2111_11103_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu
P = ctypes.c_void_p


@pytest.mark.parametrize("c", [1, 3, 40, 64, 65, 132, 300])
@pytest.mark.parametrize("agg", ["sum", "maxsum", "mul"])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_finalize_vs_oracle(c, agg, dtype):
    rng = np.random.default_rng(c * 7 + len(agg))
    n = 2003
    if agg == "mul":
        acc = -np.abs(rng.normal(size=(n, c)) * 30.0)
    else:
        acc = np.abs(rng.normal(size=(n, c)))
        acc[::17] = 0.0  # zero mass: unobserved for sum / maxsum
    acc[5, :] = acc[5, 0]  # a fully tied row: first maximum
    if c > 2:
        acc[9, 2] = np.nan  # NaN wins the argmax
    acc = acc.astype(dtype).astype(np.float64)
    counts = rng.integers(0, 3, size=n).astype(np.uint32)
    counts[5] = counts[9] = 1
    stride = (c + 3) // 4 * 4
    dev = torch.device("cuda")
    tdt = torch.float32 if dtype == "float32" else torch.float64
    a_d = torch.zeros((n, stride), dtype=tdt, device=dev)
    a_d[:, :c] = torch.as_tensor(acc, dtype=tdt)
    cnt = torch.as_tensor(counts.astype(np.int32), device=dev)
    rows = torch.empty((n, c), dtype=torch.float32, device=dev)
    unobs = torch.empty(n, dtype=torch.uint8, device=dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    N.check(N.load().tfb_finalize(P(a_d.data_ptr()), int(dtype == "float64"), stride, P(cnt.data_ptr()), n, c,
                                  N.AGG_IDS[agg], P(rows.data_ptr()), P(unobs.data_ptr()), P(labels.data_ptr()),
                                  P(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref_rows, ref_unobs = O.finalize(acc, counts.astype(np.int64), agg)
    np.testing.assert_array_equal(unobs.cpu().numpy().astype(bool), ref_unobs)
    np.testing.assert_allclose(rows.cpu().numpy(), ref_rows, rtol=1e-6, atol=1e-7)
    np.testing.assert_array_equal(labels.cpu().numpy(), O.texel_argmax(ref_rows, ref_unobs))


@pytest.mark.parametrize("c", [1, 2, 13, 40])
def test_probs_argmax_matches_numpy(c):
    """tfb_probs_argmax (the network-argmax fallback, cli.py:293): NumPy's
    first-maximum / first-NaN rule, ties and negative values included."""
    rng = np.random.default_rng(c)
    p = rng.integers(0, 4, size=(997, c)).astype(np.float32) / 3.0  # many ties
    p[::13, -1] = np.nan
    p[::29, 0] = -1.0
    p[5] = np.nan
    d = torch.as_tensor(p, device="cuda")
    out = torch.empty(len(p), dtype=torch.int32, device="cuda")
    N.check(N.load().tfb_probs_argmax(P(d.data_ptr()), len(p), c, P(out.data_ptr()),
                                      P(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), p.argmax(axis=1))

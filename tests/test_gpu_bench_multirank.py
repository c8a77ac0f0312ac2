"""bench.py's N>1 code path end to end on the one GPU a test box has: two gloo
ranks share it (``--share-gpu``, a functional check the JSON line marks as
such, never a measurement) and strong-scale the same job a single rank runs.
The labels after reduce-scatter -> slice finalize -> all-gather must match the
one-rank labels (float32 partial sums re-associate across the reduce-scatter,
so near-ties may flip: at most 1e-4 of the texels)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMMON = ["--frames", "64", "--batch", "32", "--steps", "1", "--warmup", "1", "--no-f64", "--no-e2e",
          "--no-render", "--no-cpu"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


@pytest.mark.gpu
def test_bench_two_ranks_match_one(tmp_path):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    one = tmp_path / "one.npy"
    two = tmp_path / "two.npy"
    r1 = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--dump-labels", str(one)] + COMMON,
                        capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                         "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                         "--dist-backend", "gloo", "--share-gpu", "--dump-labels", str(two)] + COMMON,
                        capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r2.returncode == 0, r2.stderr[-3000:]
    line = _last_json(r2.stdout)
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2 and "functional_test" in line
    assert line["config"]["frames_per_gpu"] == 32 and line["config"]["frames_total"] == 64
    a, b = np.load(one), np.load(two)
    assert a.shape == b.shape and a.size > 0
    assert (a >= 0).mean() > 0.5  # the job really observed most texels
    assert (a != b).mean() <= 1e-4

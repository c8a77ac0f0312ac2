"""bench.py's launch contract without a GPU: `--gpus N` under torchrun must match WORLD_SIZE
(exit 2 otherwise), and `--gpus N` outside torchrun spawns N ranks itself (which here fail
loudly: no GPU), never silently running one rank."""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, timeout=240):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def test_world_size_mismatch_exits_2():
    r = _bench(["--gpus", "2"], {"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=3" in r.stderr


def test_gpus_n_spawns_n_ranks():
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs to really run: covered by the driver's scaling run")
    r = _bench(["--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert r.returncode != 0  # fewer GPUs than ranks: both spawned ranks refuse
    out = r.stdout + r.stderr
    # both ranks print the refusal (their stderr may interleave); torchrun names the failed ranks
    assert re.search(r"2 ranks but only \d visible GPUs", out), out[-2000:]
    assert "torch.distributed" in out or "ChildFailedError" in out, out[-2000:]

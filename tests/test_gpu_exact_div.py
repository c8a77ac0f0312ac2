"""csrc/exact_div.cuh: the branch-free division fast path equals __ddiv_rn
bit for bit wherever it reports ok (2^27 operand pairs, half raw bit
patterns, half rasterizer-like magnitudes)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ddiv_try_matches_div_rn(tmp_path):
    from paper_2111_11103_b200 import build as B

    exe = str(tmp_path / "exact_div_check")
    subprocess.run([B._nvcc(), *B.ARCH, "-O3", "-std=c++17", "-I" + B.CSRC,
                    os.path.join(ROOT, "tests", "cuda", "exact_div_check.cu"), "-o", exe], check=True)
    out = subprocess.run([exe, str(1 << 27)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    fast = int(out.stdout.split("fast-path")[1].split()[0])
    assert fast > (1 << 25)  # the fast path is the common case

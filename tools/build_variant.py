"""Experiment helper: build the library with extra nvcc flags into _exp/<name>.so

    python tools/build_variant.py NAME -DFOO=1 ...
    TFB_LIB=_exp/NAME.so python bench.py ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_11103_b200 import build as B  # noqa: E402


def build_variant(name, flags):
    out = os.path.join(ROOT, "_exp", name)
    os.makedirs(out, exist_ok=True)
    objs = []
    for src in B.sources():
        obj = os.path.join(out, src.replace(".cu", ".o"))
        subprocess.run([B._nvcc(), *B.ARCH, *B.COMMON, *B.PER_FILE.get(src, []), *flags, "-c",
                        os.path.join(B.CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    lib = os.path.join(ROOT, "_exp", name + ".so")
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
    return lib


if __name__ == "__main__":
    print(build_variant(sys.argv[1], sys.argv[2:]))

"""Experiment: histograms of records per tile, covering records per pixel and
pairs per tile for the bench scene (cfg2).  Builds a -DTFB_RASTER_STATS variant
of the library into _exp/ and loads it through TFB_LIB.

    python tools/raster_stats.py [frames]
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXP = os.path.join(ROOT, "_exp")


def build_variant(flags):
    sys.path.insert(0, ROOT)
    from paper_2111_11103_b200 import build as B
    os.makedirs(EXP, exist_ok=True)
    objs = []
    for src in B.sources():
        obj = os.path.join(EXP, src.replace(".cu", ".o"))
        subprocess.run([B._nvcc(), *B.ARCH, *B.COMMON, *B.PER_FILE.get(src, []), *flags, "-c",
                        os.path.join(B.CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    lib = os.path.join(EXP, "libtexelfuse_b200_stats.so")
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
    return lib


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    lib = os.path.join(EXP, "libtexelfuse_b200_stats.so")
    if not os.path.exists(lib):
        lib = build_variant(["-DTFB_RASTER_STATS"])
    os.environ["TFB_LIB"] = lib
    sys.path.insert(0, ROOT)
    from paper_2111_11103_b200 import _native as N  # build_variant imported the package already:
    N._lib = None                                     # bind the stats variant explicitly
    N.load(lib)
    import torch
    from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    cams = random_room_trajectory(frames, scannet_intrinsics(), seed=0)
    probs = softmax_maps(1, 480, 640, 40, seed=0, device="cuda")
    ann = MeshAnnotation(mesh, layout, num_classes=40, max_batch=32)
    ann.add_batch([probs[0]] * frames, cams)
    torch.cuda.synchronize()
    L = ctypes.CDLL(lib)
    out = (ctypes.c_ulonglong * 64)()
    L.tfb_debug_raster_stats(out, 1)
    h = list(out)
    tiles = sum(h[0:16]) + h[48]
    print("frames", frames, "tiles", tiles, "big", h[48])
    print("records/tile (bucket of 32):", [round(x / tiles, 4) for x in h[0:16]])
    pix = sum(h[16:32])
    print("covering records/pixel:", [round(x / pix, 4) for x in h[16:32]])
    print("pairs/tile (bucket of 256):", [round(x / tiles, 4) for x in h[32:48]])


if __name__ == "__main__":
    main()

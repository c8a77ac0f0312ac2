"""Device time of the batched fold at cfg2 with and without the fused network-argmax
fallback output (the session caches it per frame, bindings/__init__.py:112), f32 and
fixed64 accumulators.  python tools/fallback_cost.py"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout  # noqa: E402
from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps  # noqa: E402


def main():
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    n = 1024
    frames = random_room_trajectory(n, scannet_intrinsics(), seed=0)
    pool = softmax_maps(8, 480, 640, 40, seed=0)
    probs = [pool[i % 8] for i in range(n)]
    out = {}
    fb = torch.empty((n, 480 * 640), dtype=torch.int32, device="cuda")
    for acc in ("float32", "fixed64", "float64"):
        ann = MeshAnnotation(mesh, layout, num_classes=40, aggregator="mul", accum_dtype=acc, max_batch=256)
        cams = ann.scene.cams_tensor(frames)
        for with_fb in (False, True):
            ann.profile = []
            for rep in range(2):
                ann.reset()
                ann.profile = []
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ann.add_batch(probs, cams, width=640, height=480, fallback_out=fb if with_fb else None)
                e1.record()
                torch.cuda.synchronize()
            prof, ann.profile = ann.profile, None
            fuse = sum(a.elapsed_time(b) for _, _, _, a, b in prof)
            ras = sum(a.elapsed_time(b) for _, a, b, _, _ in prof)
            out["%s%s" % (acc, "+fallback" if with_fb else "")] = {
                "frames_per_s": round(n / (e0.elapsed_time(e1) / 1000.0)), "fuse_us_per_frame": round(1000 * fuse / n, 2),
                "raster_us_per_frame": round(1000 * ras / n, 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

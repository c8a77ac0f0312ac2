"""Secondary measurements of the other BASELINE/SURVEY §8(d) configurations
(not bench lines: bench.py's headline is cfg2).  One fusion job per config,
timed with CUDA events after a warm-up job; prints one JSON line per config.

    python tools/bench_configs.py [cfg1 cfg2sum cfg4 cfg5 cfg2furn]
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2111_11103_b200 import Mesh, MeshAnnotation, uniform_layout  # noqa: E402
from paper_2111_11103_b200.geometry import Intrinsics  # noqa: E402
from paper_2111_11103_b200.synth import (make_furnished_room, make_room, random_room_trajectory,  # noqa: E402
                                         softmax_maps)

CONFIGS = {
    # name: (tess, width, height, fx, classes, frames, aggregator, layout steps, batch, pool)
    "cfg1": (32, 160, 120, 160.0, 13, 20, "sum", 1, 20, 4),
    "cfg2": (158, 640, 480, 577.87, 40, 2000, "mul", 1, 256, 8),
    "cfg2sum": (158, 640, 480, 577.87, 40, 2000, "sum", 1, 256, 8),
    "cfg4": (158, 640, 480, 577.87, 40, 2000, "mul", 8, 256, 8),
    "cfg5": (646, 1920, 1080, 1728.0, 19, 500, "mul", 1, 32, 4),  # one GPU's share of the 8-GPU job
    # cfg2 with furniture (SURVEY §7 hard part 9): 10 boxes, +1.4 % triangles, occlusion / overdraw
    "cfg2furn": (158, 640, 480, 577.87, 40, 2000, "mul", 1, 256, 8),
    # cfg2 with the float64 accumulator (the library API default, the reference's precision)
    "cfg2f64": (158, 640, 480, 577.87, 40, 2000, "mul", 1, 256, 8),
    # cfg2 with the fixed-point accumulator (the session default and deterministic=true)
    "cfg2fix": (158, 640, 480, 577.87, 40, 2000, "mul", 1, 256, 8),
    # cfg2, sum aggregator (configs[0]'s rule) with the float64 accumulator (the library default)
    "cfg2sumf64": (158, 640, 480, 577.87, 40, 2000, "sum", 1, 256, 8),
}


def run(name):
    tess, W, H, fx, c, frames, agg, steps, batch, pool = CONFIGS[name]
    t0 = time.time()
    v, t = make_furnished_room((6.0, 5.0, 3.0), tess) if name.endswith("furn") else make_room((6.0, 5.0, 3.0), tess)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, steps)
    intr = Intrinsics(fx=fx, fy=fx, cx=(W - 1) / 2.0, cy=(H - 1) / 2.0, width=W, height=H)
    cams = random_room_trajectory(frames, intr, seed=0)
    maps = softmax_maps(pool, H, W, c, seed=0, device="cuda")
    probs = [maps[i % pool] for i in range(frames)]
    order = {"1": True, "0": False}.get(os.environ.get("TFB_ORDER", ""))  # force the item order on / off
    ann = MeshAnnotation(mesh, layout, num_classes=c, aggregator=agg, weight_mode="images_iid", order_items=order,
                         accum_dtype=("float64" if name.endswith("f64") else "fixed64" if name.endswith("fix")
                                      else "float32"), max_batch=batch)
    cams_dev = ann.scene.cams_tensor(cams)
    setup_s = time.time() - t0

    def job():
        ann.reset()
        ann.add_batch(probs, cams_dev, width=W, height=H)
        ann.labels()

    job()
    torch.cuda.synchronize()
    ann.profile = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    job()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof, ann.profile = ann.profile, None
    raster = sum(r0.elapsed_time(r1) for _, r0, r1, _, _ in prof)
    fuse = sum(f0.elapsed_time(f1) for _, _, _, f0, f1 in prof)
    b_frame = H * W * (4 * c + 8)
    # the accumulator read-modify-write term, reported on its own (never folded into
    # the headline bytes): T_frame distinct texels touched per frame x stride x 4 B x 2
    touched = []
    for k in range(0, min(frames, 64), 8):
        ann.reset()
        ann.add_batch(probs[k:k + 1], cams_dev[k:k + 1], width=W, height=H)
        touched.append(int((ann.texture.counts_device() > 0).sum().item()))
    t_frame = sum(touched) / len(touched)
    print(json.dumps({
        "config": name, "triangles": mesh.num_triangles, "texels": layout.total_texels, "size": [W, H],
        "classes": c, "aggregator": agg, "frames": frames, "batch": batch,
        "frames_per_s": frames / (ms / 1000.0), "ms_per_job": ms,
        "raster_us_per_frame": 1000.0 * raster / frames, "fuse_us_per_frame": 1000.0 * fuse / frames,
        "fuse_gbs": b_frame * frames / (fuse / 1000.0) / 1e9, "setup_s": round(setup_s, 1),
        "bytes_per_frame_maps": b_frame, "texels_touched_per_frame": round(t_frame),
        "accum_rmw_bytes_per_frame": int(t_frame * ann.texture.stride * (8 if ann.texture.accum_kind else 4) * 2),
        "accum_bytes": int(layout.total_texels * ann.texture.stride * (8 if ann.texture.accum_kind else 4)),
        "order_items": ann._use_order(),
        "fuse_kernel": ("k_fuse_fast D64 (float64)" if name.endswith("f64") else
                        "k_fuse_fast fixed64" if name.endswith("fix") else
                        "k_fuse_fast<VEC>" if c % 4 == 0 else "k_fuse_fast<scalar quads>"),
    }), flush=True)
    del ann, maps, probs
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CONFIGS)):
        run(name)

"""Throughput of the reference-style per-frame APIs on cfg2 (not a bench line):
the session (open_session / add_frame / finalize_and_render) and the library
loop (rasterize -> compute_pixel_weights -> accumulate_frame), device maps.

    python tools/bench_session.py [frames]
"""
import json
import os
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2111_11103_b200 import (Mesh, MeshAnnotation, accumulate_frame, compute_pixel_weights, finalize,  # noqa: E402
                                   init_texture, rasterize, save_ply, save_trajectory, uniform_layout)
from paper_2111_11103_b200.session import add_frame, finalize_and_render, open_session  # noqa: E402
from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fixed64", "float32", "float64", "ann", "lib"]
    v, t = make_room((6.0, 5.0, 3.0), 158)
    mesh = Mesh.from_arrays(v, t)
    frames = random_room_trajectory(n, scannet_intrinsics(), seed=0)
    maps = softmax_maps(8, 480, 640, 40, seed=0)
    out = {"frames": n}
    with tempfile.TemporaryDirectory() as d:
        mp, tp = os.path.join(d, "m.ply"), os.path.join(d, "t.txt")
        save_ply(mp, mesh)
        save_trajectory(tp, frames)
        for rep, acc in enumerate(only):
            if acc not in ("fixed64", "float32", "float64"):
                continue
            s = open_session(mp, tp, 0.0, "mul", "images_iid", 40, accum_dtype=acc)
            for fr in frames[:300]:  # warm-up: the GPU leaves its idle clocks, buffers are allocated
                add_frame(s, fr.frame_id, maps[0])
            s.ann.flush()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.time()
            e0.record()
            s.ann.profile = []
            for i, fr in enumerate(frames):
                add_frame(s, fr.frame_id, maps[i % 8])
            t_py = time.time() - t0
            s.ann.flush()
            e1.record()
            torch.cuda.synchronize()
            dt = time.time() - t0
            out["s%d_%s_host_us" % (rep, acc)] = round(1e6 * t_py / n, 1)
            out["s%d_%s_device_us" % (rep, acc)] = round(1e3 * e0.elapsed_time(e1) / n, 1)
            out["s%d_%s_batch" % (rep, acc)] = s.ann._batch_for(640, 480)
            prof, s.ann.profile = s.ann.profile, None
            out["s%d_%s_raster_fuse_us" % (rep, acc)] = [
                round(1e3 * sum(a.elapsed_time(b) for _, a, b, _, _ in prof) / n, 1),
                round(1e3 * sum(a.elapsed_time(b) for _, _, _, a, b in prof) / n, 1)]
            import gc
            out["session_%s_rep%d" % (acc, rep)] = round(n / dt)
            finalize_and_render(s, [frames[0].frame_id])
            out["session_add_frame_%s%s" % (acc, " (default)" if acc == "fixed64" else "")] = round(n / dt)
            del s
            gc.collect()
    if "ann" not in only:
        print(json.dumps(out), flush=True)
        return
    ann = MeshAnnotation(mesh, uniform_layout(mesh, 1), num_classes=40, aggregator="mul")
    for fr in frames[:300]:
        ann.add(maps[0], fr)
    ann.flush()
    torch.cuda.synchronize()
    t0 = time.time()
    for i, fr in enumerate(frames):
        ann.add(maps[i % 8], fr)
    ann.labels()
    torch.cuda.synchronize()
    out["meshannotation_add_float32"] = round(n / (time.time() - t0))
    layout = uniform_layout(mesh, 1)
    tex = init_texture(layout, 40, "mul", accum_dtype="float32")
    for i, fr in enumerate(frames[:30]):  # warm-up: the layout's device scene, pinned readback buffers
        ids = rasterize(mesh, layout, fr)
        accumulate_frame(tex, ids, maps[i % 8], compute_pixel_weights(ids, "images_iid"))
    tex = init_texture(layout, 40, "mul", accum_dtype="float32")
    m = min(n, 300)
    torch.cuda.synchronize()
    t0 = time.time()
    for i, fr in enumerate(frames[:m]):
        ids = rasterize(mesh, layout, fr)
        accumulate_frame(tex, ids, maps[i % 8], compute_pixel_weights(ids, "images_iid"))
    finalize(tex)
    torch.cuda.synchronize()
    out["library_loop_float32"] = round(m / (time.time() - t0))
    out["note"] = ("wall clock, device maps (8-map pool), cfg2 scene, frames/s; library loop over %d frames "
                   "after 30 warm-up frames" % m)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

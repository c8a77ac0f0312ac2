"""Benchmark: fused frames/s of the label-fusion hot path (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1], "ScanNet-scale synthetic scene"): make_room tess=158
(299,568 triangles, 151,686 vertices), uniform_layout steps=1 (n_x = 299,568
texels), 2000 frames of 640x480 from a seeded random in-room trajectory,
c = 40 classes, softmax(N(0, 2^2)) float32 probability maps, aggregator mul
(the paper default), weights images_iid, float32 accumulator.

One step = one whole fusion job: zero the texture, rasterize + weight +
scatter-add all 2000 frames (batches of --batch frames), finalize + argmax;
with N > 1 the accumulator rows are sum-reduce-scattered (NCCL), each rank
finalizes its slice and the int32 labels are all-gathered.  `value` = frames of all
ranks / max-over-ranks device time (weak scaling: 2000 frames per GPU).
Inputs are larger than L2: the frames cycle a pool of 8 distinct maps per
GPU (8 x 49.2 MB = 393 MB > 126 MB L2), so every frame's probabilities are
streamed from HBM.

`e2e` is the same job through the public MeshAnnotation API with the
probability maps in pinned HOST memory: every step copies all 2000 maps
host→device and reads the texel labels back.

`--impl reference` times the CPU reference path (the oracle's C port of the
reference's rasterize → weights → accumulate loop, frame-parallel over all
host threads) on a bounded sample of the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W, C = 480, 640, 40
TESS = 158
FRAMES = 2000
POOL = 8
AGG = "mul"
WMODE = "images_iid"
B_FRAME = H * W * (4 * C + 8)  # algorithmic bytes per frame of the scatter-add
METRIC = "fused frames/sec (640x480, c=40)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _config(args, n):
    return {"workload": "cfg2: room 299,568 tris, %d frames/GPU 640x480, c=40, %s, %s, steps=1 layout"
                        % (args.frames, AGG, WMODE),
            "frames_per_gpu": args.frames, "triangles": 299568, "texels": 299568, "classes": C,
            "aggregator": AGG, "weights": WMODE, "accum": "float32", "batch": args.batch, "overlap": bool(args.overlap),
            "parallelism": "frame-sharded dp%d" % n,
            "l2": "inputs larger than L2: 8-map pool per GPU (393 MB) cycled, accumulator 47.9 MB"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 7:
                        rows.append(parts)
        finally:
            if self.path:
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(args, frames_sample, threads, scene=None):
    """Frames/s of the oracle's C port of the reference loop on a bounded sample."""
    import oracle as O
    from paper_2111_11103_b200.geometry import pack_camera, uniform_layout, Mesh
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics

    if scene is None:
        v, t = make_room((6.0, 5.0, 3.0), TESS)
        mesh = Mesh.from_arrays(v, t)
        layout = uniform_layout(mesh, 1)
    else:
        mesh, layout = scene
    frames = random_room_trajectory(frames_sample, scannet_intrinsics(), seed=0)
    rng = np.random.default_rng(0)
    pool = []
    for i in range(min(frames_sample, 4)):
        lg = rng.normal(scale=2.0, size=(H, W, C)).astype(np.float32)
        lg -= lg.max(axis=2, keepdims=True)
        e = np.exp(lg)
        pool.append((e / e.sum(axis=2, keepdims=True)).astype(np.float32))
    probs = [pool[i % len(pool)] for i in range(frames_sample)]
    cams = np.stack([pack_camera(f) for f in frames])
    t0 = time.perf_counter()
    acc, cnt = O.fuse_frames_c(mesh.vertices, mesh.triangles, layout.steps, layout.origins, layout.offsets,
                               layout.total_texels, cams, W, H, probs, AGG, WMODE, nthreads=threads)
    O.finalize_c(acc, cnt, AGG, want_rows=False)
    dt = time.perf_counter() - t0
    return frames_sample / dt, dt


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    threads = min(len(os.sched_getaffinity(0)), 64)
    sample = 8 * threads
    for _ in range(args.warmup):
        cpu_reference(args, threads, threads)
    vals = []
    t_total = 0.0
    for _ in range(args.steps):
        v, dt = cpu_reference(args, sample, threads)
        vals.append(v)
        t_total += dt
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args, world),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": "%d cfg2 frames per step (rasterize+images_iid+mul accumulate), "
                                       "frame-parallel C port of the reference loop over %d threads, "
                                       "plus finalize" % (sample, threads)},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2111_11103_b200 import MeshAnnotation
    from paper_2111_11103_b200.geometry import Mesh, pack_camera, uniform_layout
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)  # before the process group, so NCCL binds this rank's GPU
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)

    v, t = make_room((6.0, 5.0, 3.0), TESS)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    frames = random_room_trajectory(args.frames, scannet_intrinsics(), seed=1000 + rank)
    cams_dev = torch.as_tensor(np.stack([pack_camera(f) for f in frames])).to(dev)
    pool = softmax_maps(POOL, H, W, C, seed=rank, device=dev)
    probs_list = [pool[i % POOL] for i in range(args.frames)]
    ann = MeshAnnotation(mesh, layout, num_classes=C, aggregator=AGG, weight_mode=WMODE, accum_dtype="float32",
                         max_batch=args.batch, device=dev, overlap=args.overlap,
                         fuse_ctas_per_sm=args.fuse_ctas if args.fuse_ctas >= 0 else None)
    stream = torch.cuda.current_stream(dev)

    def step():
        ann.reset()
        ann.add_batch(probs_list, cams_dev, width=W, height=H)
        if world > 1:
            ann.finalize_distributed()  # reduce-scatter rows, finalize a slice per rank, all-gather labels
        ann.labels()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 1)):
        step()
    barrier()
    ann.profile = []
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        t_start.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
        barrier()
    prof, ann.profile = ann.profile, None
    ms = t_start.elapsed_time(t_end)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * args.frames * args.steps / (ms_max / 1000.0)

    raster_ms = sum(r0.elapsed_time(r1) for _, r0, r1, _, _ in prof)
    fuse_ms = sum(f0.elapsed_time(f1) for _, _, _, f0, f1 in prof)
    fuse_frames = sum(p_[0] for p_ in prof)
    # k_fuse launches: tfb_fuse carries at most 256 frames per launch
    n_launch_fuse = sum((p_[0] + 255) // 256 for p_ in prof)
    # our kernels per timed step: per batch k_ccull, k_ccands (k_verts, k_cull without scene clusters),
    # k_setup, k_raster, k_raster_big + the k_fuse launches (the hit-count reset is a dense torch
    # memset here), + k_finalize once
    batches = [min(args.batch, args.frames - b0) for b0 in range(0, args.frames, args.batch)]
    gpu_launches = args.steps * (sum(5 + (b + 255) // 256 for b in batches) + 1)
    peak, peak_kind = _peaks()
    achieved = B_FRAME * fuse_frames / (fuse_ms / 1000.0) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "fuse_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---- e2e through the public API with host (pinned) inputs --------------------------------
    e2e = None
    if not args.no_e2e:
        host_pool = [pool[i].cpu().pin_memory() for i in range(POOL)]
        host_list = [host_pool[i % POOL] for i in range(args.frames)]
        cams_host = [frames[i] for i in range(args.frames)]

        def e2e_step():
            ann.reset()
            ann.add_batch(host_list, cams_host)
            if world > 1:
                ann.finalize_distributed()
            return ann.labels(host=True)

        e2e_step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, args.e2e_steps))
        e0.record(stream)
        for _ in range(ksteps):
            labels_host = e2e_step()
        e1.record(stream)
        barrier()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": world * args.frames * ksteps / (float(e_ms.item()) / 1000.0), "unit": "frames/s",
               "h2d_bytes_per_step": args.frames * (H * W * C * 4 + 16 * 8),
               "d2h_bytes_per_step": int(labels_host.nbytes), "steps": ksteps,
               "api": "MeshAnnotation.add_batch(pinned host maps) + labels(host=True)"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        threads = min(len(os.sched_getaffinity(0)), 64)
        sample = 64 * threads
        val, dt = cpu_reference(args, sample, threads, scene=(mesh, layout))
        cpu = {"value": val, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": "%d cfg2 frames (rasterize+images_iid+mul accumulate+finalize), oracle C port, "
                         "frame-parallel over %d host threads, %.1f s" % (sample, threads, dt)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": _config(args, world),
            "roofline": {"bound": "hbm", "kernel": "k_fuse (tfb_fuse)", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "bytes_per_frame": B_FRAME,
                         "launch_ms_avg": fuse_ms / max(n_launch_fuse, 1),
                         "frames_per_launch": fuse_frames / max(n_launch_fuse, 1)},
            "breakdown_ms_per_step": {"raster": raster_ms / args.steps, "fuse": fuse_ms / args.steps,
                                      "other": ms_max / args.steps - (raster_ms + fuse_ms) / args.steps},
            "clocks": clocks.summary(), "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": gpu_launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--overlap", type=int, default=0)
    ap.add_argument("--fuse-ctas", type=int, default=-1, help="cap on resident scatter-add CTAs per SM (-1: auto)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

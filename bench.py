"""Benchmark: fused frames/s of the label-fusion hot path (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1], "ScanNet-scale synthetic scene"): make_room tess=158
(299,568 triangles, 151,686 vertices), uniform_layout steps=1 (n_x = 299,568
texels), 2000 frames of 640x480 from a seeded random in-room trajectory,
c = 40 classes, softmax(N(0, 2^2)) float32 probability maps, aggregator mul
(the paper default), weights images_iid, float32 accumulator.

One step = one whole fusion job: zero the texture, rasterize + weight +
scatter-add the rank's frames (batches of --batch frames), finalize + argmax;
with N > 1 the accumulator rows are sum-reduce-scattered (NCCL), each rank
finalizes its slice and the int32 labels are all-gathered.  `value` = frames of all
ranks / max-over-ranks device time.  --scaling strong (default; BASELINE
configs[2]: "same ScanNet-scale scene frame-sharded at 2/4/8 B200") splits the
2000-frame trajectory into N contiguous blocks; --scaling weak gives every
rank its own 2000 frames.

Multi-GPU: `python bench.py --gpus N` re-executes itself under
torch.distributed.run with N ranks (one per GPU) unless it already runs under
torchrun, in which case WORLD_SIZE must equal N (exit code 2 otherwise).
Inputs are larger than L2: the frames cycle a pool of 8 distinct maps per
GPU (8 x 49.2 MB = 393 MB > 126 MB L2), so every frame's probabilities are
streamed from HBM.

`e2e` is the same job through the public MeshAnnotation API with the
probability maps in pinned HOST memory: every step copies all 2000 maps
host→device and reads the texel labels back.

`--impl reference` times the CPU reference path (the oracle's C port of the
reference's rasterize → weights → accumulate → finalize loop, frame-parallel
over all host threads, parallel reduction and finalize) on a bounded sample
of the same workload: exactly the function and sample size of the
`cpu_baseline` leg, so the two agree.
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


def _frames_per_rank(args, n):
    return args.frames if args.scaling == "weak" else -(-args.frames // n)


def _config(args, n):
    total = args.frames * (n if args.scaling == "weak" else 1)
    return {"workload": "cfg%s: room 299,568 tris, %d frames 640x480 (%s scaling over %d GPU), c=40, %s, %s, "
                        "steps=1 layout" % ("2" if n == 1 else "3", total, args.scaling, n, AGG, WMODE),
            "frames_total": total, "frames_per_gpu": _frames_per_rank(args, n), "scaling": args.scaling,
            "triangles": 299568, "texels": 299568, "classes": C,
            "aggregator": AGG, "weights": WMODE, "accum": "float32", "batch": args.batch, "overlap": bool(args.overlap),
            "split_raster": args.split_raster == 1 or (args.split_raster < 0 and os.environ.get("TFB_SPLIT_RASTER") == "1"),
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


CPU_FRAMES_PER_THREAD = 32  # bounded sample: ~3-6 s of CPU work per sample on 16-64 threads


def _host_cpu():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model}


def _cpu_threads():
    return min(len(os.sched_getaffinity(0)), 64)


def _cpu_sample_desc(sample, threads, dt=None):
    return ("%d cfg2 frames (rasterize + images_iid weights + mul accumulate into float64, then finalize + "
            "argmax), oracle C port of the reference loop, frame-parallel over %d host threads with a "
            "row-parallel reduction%s" % (sample, threads, "" if dt is None else ", %.1f s" % dt))


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    world = max(world, args.gpus)
    threads = _cpu_threads()
    sample = CPU_FRAMES_PER_THREAD * threads
    from paper_2111_11103_b200.geometry import Mesh, uniform_layout
    from paper_2111_11103_b200.synth import make_room

    v, t = make_room((6.0, 5.0, 3.0), TESS)
    mesh = Mesh.from_arrays(v, t)
    scene = (mesh, uniform_layout(mesh, 1))
    for _ in range(args.warmup):
        cpu_reference(args, threads, threads, scene=scene)
    vals = []
    t_total = 0.0
    for _ in range(args.steps):
        val, dt = cpu_reference(args, sample, threads, scene=scene)
        vals.append(val)
        t_total += dt
    value = statistics.median(vals)
    cfg = _config(args, world)
    cfg["reference_sample_frames_per_step"] = sample
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / max(args.steps, 1),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg, "host_cpu": _host_cpu(),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": _cpu_sample_desc(sample, threads) + " per step"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2111_11103_b200 import MeshAnnotation
    from paper_2111_11103_b200.dist import shard_bounds
    from paper_2111_11103_b200.geometry import Mesh, pack_camera, uniform_layout
    from paper_2111_11103_b200.synth import make_room, random_room_trajectory, scannet_intrinsics, softmax_maps

    world, rank, local = _dist_env()
    if world > torch.cuda.device_count() and not args.share_gpu:
        raise SystemExit("bench.py: %d ranks but only %d visible GPUs" % (world, torch.cuda.device_count()))
    if args.share_gpu:  # functional self-test of the multi-rank code path only (never a measurement)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)  # before the process group, so NCCL binds this rank's GPU
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend, init_method="env://")
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)  # forces communicator creation; every rank must contribute
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(), "nranks_seen": int(probe.item()),
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())}
        if int(probe.item()) != world:
            raise SystemExit("bench.py: NCCL communicator saw %d ranks, expected %d" % (int(probe.item()), world))

    v, t = make_room((6.0, 5.0, 3.0), TESS)
    mesh = Mesh.from_arrays(v, t)
    layout = uniform_layout(mesh, 1)
    if args.scaling == "weak":
        lo = 0
        frames = random_room_trajectory(args.frames, scannet_intrinsics(), seed=1000 + rank)
    else:  # strong: one 2000-frame trajectory, contiguous block per rank (dist.shard_bounds)
        lo, hi = shard_bounds(args.frames, rank, world)
        frames = random_room_trajectory(args.frames, scannet_intrinsics(), seed=1000)[lo:hi]
    nf = len(frames)
    cams_dev = torch.as_tensor(np.stack([pack_camera(f) for f in frames])).to(dev)
    # strong scaling: frame g gets map g % POOL whatever the rank count, so every N fuses the same job
    pool = softmax_maps(POOL, H, W, C, seed=rank if args.scaling == "weak" else 0, device=dev)
    probs_list = [pool[(lo + i) % POOL] for i in range(nf)]
    ann = MeshAnnotation(mesh, layout, num_classes=C, aggregator=AGG, weight_mode=WMODE, accum_dtype="float32",
                         max_batch=args.batch, device=dev, overlap=args.overlap,
                         fuse_ctas_per_sm=args.fuse_ctas if args.fuse_ctas >= 0 else None,
                         split_raster=None if args.split_raster < 0 else bool(args.split_raster))
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
    if args.dump_labels and rank == 0:  # after the timed region: the fused labels, for cross-N checks
        np.save(args.dump_labels, ann.labels(host=True))
    ms = t_start.elapsed_time(t_end)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    frames_t = torch.tensor([float(nf)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(frames_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    frames_all = int(frames_t.item())
    value = frames_all * args.steps / (ms_max / 1000.0)

    raster_ms = sum(r0.elapsed_time(r1) for _, r0, r1, _, _ in prof)
    fuse_ms = sum(f0.elapsed_time(f1) for _, _, _, f0, f1 in prof)
    fuse_frames = sum(p_[0] for p_ in prof)
    # k_fuse launches: tfb_fuse carries at most 256 frames per launch
    n_launch_fuse = sum((p_[0] + 255) // 256 for p_ in prof)
    # our kernels per timed step: per batch k_ccull, k_ccsetup, k_raster<64>, k_raster_tier<128>,
    # k_raster_big + the k_fuse launches (the hit-count reset is a dense torch memset here),
    # + k_finalize once
    batches = [min(args.batch, nf - b0) for b0 in range(0, nf, args.batch)]
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

    # ---- secondary: the same job with the float64 accumulator (the reference's arithmetic) ----
    f64 = None
    if not args.no_f64:
        ann64 = MeshAnnotation(mesh, layout, num_classes=C, aggregator=AGG, weight_mode=WMODE,
                               accum_dtype="float64", max_batch=args.batch, device=dev)

        def step64():
            ann64.reset()
            ann64.add_batch(probs_list, cams_dev, width=W, height=H)
            if world > 1:
                ann64.finalize_distributed()
            ann64.labels()

        step64()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        step64()
        a1.record(stream)
        barrier()
        f_ms = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(f_ms, op=dist.ReduceOp.MAX)
        f64 = {"value": frames_all / (float(f_ms.item()) / 1000.0), "unit": "frames/s", "steps": 1,
               "accum": "float64 (atomicAdd f64; the reference's accumulator precision)"}
        del ann64

    # ---- e2e through the public API with host (pinned) inputs --------------------------------
    e2e = None
    if not args.no_e2e:
        host_pool = [pool[i].cpu().pin_memory() for i in range(POOL)]
        host_list = [host_pool[i % POOL] for i in range(nf)]
        cams_host = [frames[i] for i in range(nf)]

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
        e2e = {"value": frames_all * ksteps / (float(e_ms.item()) / 1000.0), "unit": "frames/s",
               "h2d_bytes_per_step": nf * (H * W * C * 4 + 16 * 8),
               "d2h_bytes_per_step": int(labels_host.nbytes), "steps": ksteps,
               "api": "MeshAnnotation.add_batch(pinned host maps) + labels(host=True)",
               "note": "bytes per rank; every rank copies its own frames"}
        if not args.no_pageable:
            # the reference API's natural input: pageable NumPy maps (one step, a bounded
            # 256-frame sample: every map is staged through the driver's pageable copy path)
            np_pool = [host_pool[i].numpy().copy() for i in range(POOL)]  # ordinary (pageable) host memory
            m = min(nf, 256)

            def pageable_step():
                ann.reset()
                ann.add_batch([np_pool[i % POOL] for i in range(m)], cams_host[:m])
                return ann.labels(host=True)

            pageable_step()
            barrier()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            pageable_step()
            p1.record(stream)
            barrier()
            p_ms = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(p_ms, op=dist.ReduceOp.MAX)
            e2e["pageable_numpy"] = {"value": world * m / (float(p_ms.item()) / 1000.0), "unit": "frames/s",
                                     "frames_per_rank": m,
                                     "api": "MeshAnnotation.add_batch(list of pageable np.ndarray) + labels(host=True)"}

    # ---- re-render throughput (reported separately): rasterize + label gather
    render = None
    if not args.no_render:
        ann.reset()
        ann.add_batch(probs_list, cams_dev, width=W, height=H)
        ann.labels()
        out_imgs = ann.render(cams_dev, width=W, height=H)
        del out_imgs  # the timed call reuses this allocation instead of growing the pool inside the timing
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        out_imgs = ann.render(cams_dev, width=W, height=H)
        q1.record(stream)
        barrier()
        q_ms = torch.tensor([q0.elapsed_time(q1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(q_ms, op=dist.ReduceOp.MAX)
        render = {"value": frames_all / (float(q_ms.item()) / 1000.0), "unit": "frames/s",
                  "api": "MeshAnnotation.render(cameras) -> (B, H, W) int32 labels on the device "
                         "(renderback.py:28-56 per frame: rasterize + per-pixel texel-label gather)"}
        del out_imgs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        threads = _cpu_threads()
        sample = CPU_FRAMES_PER_THREAD * threads
        val, dt = cpu_reference(args, sample, threads, scene=(mesh, layout))
        cpu = {"value": val, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": _cpu_sample_desc(sample, threads, dt), "host_cpu": _host_cpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(args, world),
            "roofline": {"bound": "hbm", "kernel": "k_fuse (tfb_fuse)", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "frac_vs_8tbs_nominal": achieved / 8000.0,
                         "bytes_per_frame": B_FRAME,
                         "launch_ms_avg": fuse_ms / max(n_launch_fuse, 1),
                         "frames_per_launch": fuse_frames / max(n_launch_fuse, 1)},
            "breakdown_ms_per_step": {"raster": raster_ms / args.steps, "fuse": fuse_ms / args.steps,
                                      "other": ms_max / args.steps - (raster_ms + fuse_ms) / args.steps},
            "clocks": clocks.summary(), "e2e": e2e, "f64_accumulator": f64, "render": render, "cpu_baseline": cpu,
            "gpu_launches": gpu_launches, "comm": comm,
        }
        if args.share_gpu:
            line["functional_test"] = "ranks shared %d GPU(s) over %s: a code-path check, not a measurement" % (
                torch.cuda.device_count(), args.dist_backend)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn_ranks(args):
    """Re-execute this script under torch.distributed.run with --gpus ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator size / NVLS selection visible in the log
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES, help="trajectory length (per rank with --scaling weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--overlap", type=int, default=0)
    ap.add_argument("--split-raster", type=int, default=-1,
                    help="1: batch k+1's cull/setup/binning on a side stream under batch k's scatter-add "
                         "(-1: MeshAnnotation's default, off unless TFB_SPLIT_RASTER=1)")
    ap.add_argument("--fuse-ctas", type=int, default=-1, help="cap on resident scatter-add CTAs per SM (-1: auto)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f64", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional tests of the multi-rank path only")
    ap.add_argument("--dump-labels", default=None, help="rank 0 saves the fused labels (.npy) after the timed steps")
    ap.add_argument("--share-gpu", action="store_true",
                    help="functional test: more ranks than GPUs (ranks share them); never a measurement")
    ap.add_argument("--no-pageable", action="store_true")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0:  # not under torchrun
        if args.gpus > 1 and args.impl == "ours":
            sys.exit(_spawn_ranks(args))
        os.environ.setdefault("WORLD_SIZE", "1")
    elif world != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world), file=sys.stderr)
        sys.exit(2)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

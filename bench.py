#!/usr/bin/env python
"""Benchmark of the POTR removal-effect scoring pass on B200.

Metric (BASELINE.json): removal-effect scoring Mpix.views/s -- one step is one
full prune-score pass (forward_stats with targets, rasterizer.py:311-352) over
every view of the configuration: `value` = S*W*H / 1e6 / step seconds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU arm (oracle port, all host cores)

Workload: BASELINE config 3 -- synthetic 3M-splat shell (fixture.shell_splats,
seed 0), 200-view ring at 1237x822 -- view-sharded over the ranks (strong
scaling: the total work is the config).  The scored state is the fixture with
opacities x0.97 against the unperturbed renders as targets, so both terms of
dSE are live.  Inputs (1.4 GB of splats, 4.9 GB of targets) exceed the 126 MB
L2, so no flush is needed between steps.

One JSON line on rank 0; see DESIGN.md section "Measurement" for the keys.
"""

import argparse
import ctypes
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

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
METRIC = "removal-effect scoring Mpix·views/s"
SH_LAMBDA = 1e-12  # the s/scene SH recompute's luminance ridge (see scene_measure)
UNIT = "Mpix·views/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-scene", action="store_true", help="skip the s/scene measurement")
    ap.add_argument("--no-prune48", action="store_true",
                    help="skip the 48-iteration run_pruning timing")
    ap.add_argument("--cpu-threads", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                    power.append(float(parts[3]))
                except ValueError:
                    continue
                for name, val in zip(self.NAMES, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def load_peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        return p, "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback"


# Work model of the fused raster + removal-effect kernel: SURVEY.md section 8(d),
# per view W = 24 E + 37 M lane-ops + 2 E exp, an fp64 exp costing ~20 DFMA
# ("fp64 parity mode"), i.e. W = 64 E + 37 M FP64 lane-ops (FMA = 1), with
#   E = bbox pixel evaluations of the reference loop (rasterizer.py:159-166),
#   M = composited contributions (:170-201).
OPS_PER_E = 24 + 2 * 20
OPS_PER_M = 37


def load_traffic(views_per_launch, config):
    """DRAM bytes (read + write) per k_raster<kScore> launch from the committed
    `ncu --set full` capture summaries (profiles/raster_traffic.json), for a
    configuration that was captured only; (None, note) otherwise."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "raster_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        c = t.get("configs", {}).get(config)
        if c is None:
            return None, f"no capture for {config} in profiles/raster_traffic.json"
        per_view = float(c["dram_bytes_per_launch"]) / float(c["views_per_launch"])
        return per_view * views_per_launch, c.get("source")
    except (OSError, ValueError, KeyError):
        return None, None


def fp64_peak_lane_ops(peaks):
    """FP64 FMA lanes per second (T/s): the DFMA microbenchmark measured on this
    pool (tools/fp64_peak.cu -> profiles/r2_fp64_peak.json), else the nominal
    148 SMs x 64 lanes x the max SM clock.  Returns (peak, source)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "r2_fp64_peak.json")
    try:
        with open(path) as f:
            return float(json.load(f)["fp64_fma_tera_per_s"]), \
                "measured: tools/fp64_peak.cu DFMA microbenchmark (profiles/r2_fp64_peak.json)"
    except (OSError, ValueError, KeyError):
        return 148 * 64 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12, \
            "nominal FP64 CUDA-core rate at sm_max_mhz (148 SMs x 64 lanes/clk)"


# ---------------------------------------------------------------------------
# the reference arm: the oracle port of the reference's CPU implementation


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2601_14821_b200.fixture import CONFIGS, config_scene
    cfg = CONFIGS[args.config]
    splats, cams = config_scene(args.config)
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    cores = host_cores()
    threads = args.cpu_threads or max(1, min(cores, int(mem_available_gb() // 4), 16))
    P = cfg["width"] * cfg["height"]
    # one step = a bounded sample of `threads` views (the reference's own
    # ThreadPoolExecutor-over-cameras parallelism, rasterizer.py:304-308)
    sample = max(1, min(threads, cfg["views"]))
    t0 = time.perf_counter()
    targets = O_render_parallel(O, splats, cams[:sample], threads)
    t_targets = time.perf_counter() - t0
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.forward_stats(pert, cams[:sample], targets, threads=threads)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    ms = 1000.0 * float(np.mean(times))
    value = sample * P / 1e6 / (ms / 1000.0)
    desc = (f"{sample} of {cfg['views']} views of {args.config} per step, "
            f"{threads} threads (oracle port of rasterizer.py forward_stats)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc, "host_cores": cores, "targets_s": t_targets},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def O_render_parallel(O, splats, cams, threads):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda c: O.render(splats, c)[0], cams))


def cpu_baseline(args, splats_pert, cams, targets_host, P):
    """Oracle port timed on this host (rank 0, N=1): a bounded sample of views."""
    from oracle import oracle as O
    cores = host_cores()
    threads = args.cpu_threads or max(1, min(cores, int(mem_available_gb() // 4), 16))
    sample = max(1, min(threads, len(cams)))
    t0 = time.perf_counter()
    O.forward_stats(splats_pert, cams[:sample], targets_host[:sample], threads=threads)
    dt = time.perf_counter() - t0
    return {"value": sample * P / 1e6 / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} views of {args.config} in {dt:.1f} s, {threads} threads",
            "host_cores": cores}


def config_dict(args, world):
    from paper_2601_14821_b200.fixture import CONFIGS
    c = CONFIGS[args.config]
    return {"workload": f"{args.config}: prune-score pass, {c['splats']} splats, "
                        f"{c['views']} views at {c['width']}x{c['height']}",
            "splats": c["splats"], "views": c["views"],
            "resolution": [c["width"], c["height"]], "parallelism": f"view-sharded x{world}",
            "l2": l2_note(c), "state": "opacity x0.97 vs unperturbed targets"}


def l2_note(c):
    """The L2 rule: inputs larger than the 126 MB L2 between timed steps, or a flush."""
    splat_gb = c["splats"] * 59 * 8 / 1e9
    target_gb = c["views"] * c["width"] * c["height"] * 3 * 8 / 1e9
    big = (splat_gb + target_gb) * 1e3 > 126
    return (f"inputs {'>' if big else '<='} L2: splats {splat_gb:.2f} GB + targets "
            f"{target_gb:.2f} GB read every step" + (", no flush" if big else
                                                    " (below L2: not a valid timing config)"))


# ---------------------------------------------------------------------------
# our arm


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    if "POTR_BENCH_DEVICE" in os.environ:  # ranks sharing one GPU (with the gloo backend)
        local = int(os.environ["POTR_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # gloo only to exercise the multi-rank logic on fewer GPUs than ranks
        backend = os.environ.get("POTR_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2601_14821_b200 import device as D
    from paper_2601_14821_b200 import distributed, rasterizer, compaction
    from paper_2601_14821_b200.fixture import CONFIGS, config_scene

    cfg = CONFIGS[args.config]
    S, W, H = cfg["views"], cfg["width"], cfg["height"]
    P = W * H
    Pv = S * P

    splats, cams = config_scene(args.config)
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    lo, hi = distributed.shard_range(S, rank, world)
    my_cams = cams[lo:hi]

    ctx = D.context()
    stream = torch.cuda.current_stream()
    ds_ref = D.DeviceSplats.from_host(splats, dev)
    ds = D.DeviceSplats.from_host(pert, dev)
    n = ds.n

    # targets of this rank's views, rendered on the GPU and kept resident
    tg = rasterizer.render_targets_device(ds_ref, my_cams)
    del ds_ref
    tptr = (ctypes.c_void_p * max(1, len(tg)))(*[t.data_ptr() for t in tg])
    cam_arr = _native_cams(my_cams)
    imp = torch.zeros(n, dtype=torch.float64, device=dev)
    dm = torch.zeros(n, dtype=torch.float64, device=dev)
    mse = torch.zeros(1, dtype=torch.float64, device=dev)
    ci = torch.empty((max(1, hi - lo), n), dtype=torch.float64, device=dev)

    if world > 1:  # per-view rows for the ordered (GPU-count-invariant) reduction
        dm_rows = torch.empty((max(1, hi - lo), n), dtype=torch.float64, device=dev)
        mse_rows = torch.empty(max(1, hi - lo), dtype=torch.float64, device=dev)

    def step():
        if world == 1:
            imp.zero_()
            dm.zero_()
            mse.zero_()
            ctx.call("potr_score_views", ctypes.byref(ds.struct()), hi - lo, cam_arr, tptr,
                     D.ptr(imp), D.ptr(ci), D.ptr(dm), D.ptr(mse))
            ctx.call("potr_finalize_stats", ctypes.c_int64(n), S, D.ptr(imp), D.ptr(dm),
                     D.ptr(mse))
            return
        # view-sharded: rows of this rank's views, then the ordered chain
        # 0 -> 1 -> ... -> W-1 + broadcast (distributed.ordered_reduce)
        ctx.call("potr_score_views_rows", ctypes.byref(ds.struct()), hi - lo, cam_arr, tptr,
                 D.ptr(ci), D.ptr(dm_rows), D.ptr(mse_rows))
        acc = distributed.ordered_reduce(ci[:hi - lo], dm_rows[:hi - lo], mse_rows[:hi - lo], n)
        distributed.finalize_sums(acc, n, S)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # work counters for the roofline (one untimed pass)
    ctx.counters(True)
    step()
    counts = ctx.counters_read()
    ctx.counters(False)

    if os.environ.get("POTR_PROFILE_STEP"):
        # one step bracketed for `ncu --profile-from-start off` (launch list of the step)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        step()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = ctx.launches()
    clocks = ClockSampler(local)
    clocks.start()
    ctx.profile(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    prof = ctx.profile_read()
    ctx.profile(False)
    clk = clocks.stop()
    launches = ctx.launches() - launches0
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
        distributed.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = Pv / 1e6 / (ms / 1000.0)

    # roofline of the dominant kernel: fused raster + removal effect
    peaks, peak_src = load_peaks()
    raster_ms, raster_n = prof["raster"]
    step_ms_sum = sum(v[0] for v in prof.values())
    E, E_live, M, K = counts
    views_here = max(1, hi - lo)
    views_per_launch = views_here / max(1, raster_n / args.steps)
    ops_per_launch = (E * OPS_PER_E + M * OPS_PER_M) / views_here * views_per_launch
    raster_avg_ms = raster_ms / max(1, raster_n)
    achieved = ops_per_launch / (raster_avg_ms / 1000.0) / 1e12
    peak, peak_note = fp64_peak_lane_ops(peaks)
    traffic, traffic_src = load_traffic(views_per_launch, args.config)
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "k_raster<kScore>",
                "unit_note": "FP64 lane-operations per second, FMA = 1 (SURVEY.md 8(d) model: "
                             "W = 24E + 37M + 2E exp at 20 DFMA each, per view)",
                "peak_source": peak_note + "; MEASURED_PEAKS.json has only HBM and bf16 "
                               "tensor peaks",
                "views_per_launch": views_per_launch,
                "raster_share_of_step": raster_ms / step_ms_sum if step_ms_sum else None,
                "per_view": {"E_bbox_evals": E / views_here, "E_live": E_live / views_here,
                             "M_contributions": M / views_here, "tile_pairs": K / views_here},
                "stage_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()}}

    # ---- end to end through the public API with host buffers -------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(args, rank, world, local, pert, cams, tg, S, Pv, dev)

    scene = None
    if not args.no_scene:
        scene = scene_measure(args, world, ds, cams, my_cams, tptr, cam_arr, lo, hi, ctx, dev,
                              splats, S)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        targets_host = [t.cpu().numpy() for t in tg[:16]]
        cpu = cpu_baseline(args, pert, cams, targets_host, P)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (fixture.shell_splats seed 0, camera ring)",
            "config": config_dict(args, world), "gpu_launches": launches,
            "clocks": clk, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "scene_seconds": scene, "peaks_source": peak_src,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _native_cam(cam):
    from paper_2601_14821_b200 import _native
    return _native.camera_struct(cam)


def _native_cams(cams):
    from paper_2601_14821_b200 import _native
    return _native.camera_array(cams)


def e2e_measure(args, rank, world, local, pert, cams, tg, S, Pv, dev):
    """compute_delta_mse through the public API every step: host splats in
    (uploaded inside the timed region), host scores out.  Two sources:
    `pageable` -- plain numpy arrays, as the reference controller hands over a
    fresh subset() every iteration (pruning.py:161; the headline e2e) -- and
    `pinned`.  Targets are the fixed reference renders, read-only host arrays
    that the API keeps resident after the first call (rasterizer.py:375-376
    semantics; see device.TargetCache)."""
    import torch
    import torch.distributed as dist
    from paper_2601_14821_b200 import distributed, rasterizer
    from paper_2601_14821_b200.scene import Splats

    def pinned_copy(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    fields = ("positions", "sh", "opacities", "scales", "rotations")
    lo, hi = distributed.shard_range(S, rank, world)
    # full-length target list; only this rank's entries are read when sharded
    targets = [None] * S
    for i, t in enumerate(tg):
        h = t.cpu().numpy()
        h.flags.writeable = False
        targets[lo + i] = h
    for s_ in range(S):
        if targets[s_] is None:
            targets[s_] = np.zeros((1, 1, 3))  # never read on this rank
    distributed.enable_view_sharding(world > 1)
    res = {}
    for kind in ("pageable", "pinned"):
        if kind == "pageable":
            host = Splats(*(np.array(getattr(pert, f), dtype=np.float64, copy=True)
                            for f in fields))
        else:
            host = Splats(*(pinned_copy(np.asarray(getattr(pert, f))) for f in fields))
        if world == 1:
            call = lambda: rasterizer.forward_stats(host, cams, targets)  # noqa: E731
        else:
            call = lambda: distributed.forward_stats_sharded(host, cams, targets)  # noqa: E731
        # warm-up mirrors the timed loop: the previous result stays alive while
        # the next call runs
        st = None
        for _ in range(max(2, args.warmup)):
            st = call()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st = call()
            _ = st.delta_mse[0]  # host result in hand
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.steps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            distributed.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        res[kind] = dt
        del st
    h2d = sum(np.asarray(getattr(pert, f)).nbytes for f in fields)
    n = len(pert.positions)
    dt = res["pageable"]
    return {"value": Pv / 1e6 / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(8 * (2 * n + 1)), "ms_per_step": dt * 1000.0,
            "source_memory": "pageable numpy arrays (the reference controller's subset())",
            "pinned": {"value": Pv / 1e6 / res["pinned"], "ms_per_step": res["pinned"] * 1e3},
            "api": "paper_2601_14821_b200.rasterizer.forward_stats (compute_delta_mse body)",
            "note": "splats uploaded every step (pageable: potr_copy_to_device's pinned ring); "
                    "targets resident after the first call (fixed, read-only); "
                    "camera_importance stays in HBM"}


def scene_measure(args, world, ds, cams, my_cams, tptr, cam_arr, lo, hi, ctx, dev, splats, S):
    """POTR end-to-end s/scene: target renders + one prune-score
    pass (with per-camera importance) + SH recompute, device-resident."""
    import torch
    import torch.distributed as dist
    from paper_2601_14821_b200 import _native
    from paper_2601_14821_b200 import device as D
    from paper_2601_14821_b200.fixture import CONFIGS
    cfg = CONFIGS[args.config]
    H, W = cfg["height"], cfg["width"]
    n = ds.n
    ds0 = D.DeviceSplats.from_host(splats, dev)
    imgs = [torch.empty((H, W, 3), dtype=torch.float64, device=dev) for _ in my_cams]
    tp = (ctypes.c_void_p * max(1, len(imgs)))(*[t.data_ptr() for t in imgs])
    imp = torch.zeros(n, dtype=torch.float64, device=dev)
    dm = torch.zeros(n, dtype=torch.float64, device=dev)
    mse = torch.zeros(1, dtype=torch.float64, device=dev)
    ci = torch.empty((max(1, hi - lo), n), dtype=torch.float64, device=dev)
    neq = torch.empty((_native.NEQ_STRIDE, n), dtype=torch.float64, device=dev)
    rgb = torch.empty((n, 3, 16), dtype=torch.float64, device=dev)
    yc = torch.empty((n, 3, 16), dtype=torch.float64, device=dev)
    status = torch.empty(n, dtype=torch.int8, device=dev)
    if world > 1:
        from paper_2601_14821_b200 import distributed
        rank = dist.get_rank()
        c0, c1 = distributed.shard_range(n, rank, world)
        nmax = max(distributed.shard_range(n, r, world)[1] - distributed.shard_range(n, r, world)[0]
                   for r in range(world))
        neq_s = torch.empty((_native.NEQ_STRIDE, max(nmax, 1)), dtype=torch.float64, device=dev)
        rgb_s = torch.empty((max(nmax, 1), 3, 16), dtype=torch.float64, device=dev)
        yc_s = torch.empty((max(nmax, 1), 3, 16), dtype=torch.float64, device=dev)
        status_s = torch.empty(max(nmax, 1), dtype=torch.int8, device=dev)
        pack = torch.zeros((max(nmax, 1), 96), dtype=torch.float64, device=dev)
        gathered = torch.empty(world * max(nmax, 1) * 96, dtype=torch.float64, device=dev)
        all_cams = _native_cams(cams)

    def run(fused):
        t = {}
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        iptr = (ctypes.c_void_p * max(1, len(imgs)))(*[t.data_ptr() for t in imgs])
        imp.zero_(), dm.zero_(), mse.zero_()
        if fused:  # targets + the first prune-score pass in one walk (potr_score_views_self)
            ctx.call("potr_score_views_self", ctypes.byref(ds0.struct()), hi - lo, cam_arr, iptr,
                     D.ptr(imp), D.ptr(ci), D.ptr(dm), D.ptr(mse))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
        else:
            ctx.call("potr_render_batch", ctypes.byref(ds0.struct()), len(my_cams),
                     _native_cams(my_cams), iptr, None)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ctx.call("potr_score_views", ctypes.byref(ds0.struct()), hi - lo, cam_arr, tp,
                     D.ptr(imp), D.ptr(ci), D.ptr(dm), D.ptr(mse))
        if world > 1:
            red = torch.cat([imp, dm, mse])
            distributed.all_reduce(red)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if world == 1:
            ctx.call("potr_sh_normal_equations", ctypes.byref(ds0.struct()), hi - lo, cam_arr,
                     D.ptr(ci), D.ptr(neq))
            ctx.call("potr_sh_solve", ctypes.byref(ds0.struct()), D.ptr(neq),
                     ctypes.c_double(SH_LAMBDA), ctypes.c_double(0.8175744761936437),
                     ctypes.c_double(0.5 / 51.0), D.ptr(rgb), D.ptr(yc), D.ptr(status))
        else:
            # splat-sharded (distributed.compact_scene_sharded on device
            # tensors): the all-to-all of camera_importance columns, this
            # rank's splat span accumulated over every view and solved, one
            # all-gather of the coefficients
            ci_s = distributed.transpose_to_splat_shard(ci[:hi - lo], S, n)
            ns = c1 - c0
            sub = D.DeviceSplats(ds0.positions[c0:c1], ds0.sh[c0:c1], ds0.opacities[c0:c1],
                                 ds0.scales[c0:c1], ds0.rotations[c0:c1])
            ctx.call("potr_sh_normal_equations", ctypes.byref(sub.struct()), S, all_cams,
                     D.ptr(ci_s), D.ptr(neq_s))
            ctx.call("potr_sh_solve", ctypes.byref(sub.struct()), D.ptr(neq_s),
                     ctypes.c_double(SH_LAMBDA), ctypes.c_double(0.8175744761936437),
                     ctypes.c_double(0.5 / 51.0), D.ptr(rgb_s), D.ptr(yc_s), D.ptr(status_s))
            pack[:ns, :48] = rgb_s[:ns].reshape(ns, 48)
            pack[:ns, 48:] = yc_s[:ns].reshape(ns, 48)
            distributed._all_gather(gathered, pack.reshape(-1), None)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        t = torch.tensor([t1 - t0, t2 - t1, t3 - t2], dtype=torch.float64, device=dev)
        if world > 1:
            distributed.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    run(False)  # warm
    parts = run(False)
    ac = float((yc[:, :, 1:] == 0).double().mean().item()) if world == 1 else \
        float((gathered.reshape(world, -1, 96)[:, :, 48:].reshape(-1, 3, 16)[:, :, 1:] == 0)
              .double().mean().item())  # (padding rows included: an estimate)
    fused = run(True)
    out = {"total_s": sum(fused), "targets_and_prune_score_s": fused[0],
           "sh_recompute_s": fused[2],
           "separate_passes": {"total_s": sum(parts), "render_targets_s": parts[0],
                               "prune_score_s": parts[1], "sh_recompute_s": parts[2]},
           "note": "total_s: the targets are rendered by the same walk that scores them "
                   "(potr_score_views_self, bit-identical to render_targets + "
                   "compute_delta_mse); separate_passes: the two calls one after the other",
           "lambda_y": SH_LAMBDA, "ac_sparsity": ac,
           "lambda_note": "lambda_y = 1e-12: AC sparsity 0.937 at C3, inside the paper's 0.70-0.97 "
                          "range (1e-7 zeroes every AC term at this importance scale; "
                          "profiles/r2_c4_report.json has 1e-11 / 1e-13)"}
    if world == 1 and not args.no_prune48:
        out.update(prune48_measure(splats, cams, imgs))
    return out


def prune48_measure(splats, cams, targets_dev):
    """The encoder's pruning stage ("48-iteration run_pruning"):
    pruning.run_pruning at q = 0.5 (delta_mse_max = 10^-9.8) through the public
    API from host splats, with the device-resident controller; targets are the
    fixed renders already in HBM."""
    import torch
    from paper_2601_14821_b200 import pruning
    cfg = pruning.PruneConfig(delta_mse_max=10.0 ** (-8.8 - 2.0 * 0.5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pruned, kept, reports = pruning.run_pruning(splats, cams, targets_dev, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"prune48_s": dt, "prune48_iterations": len(reports),
            "prune48_kept": int(len(kept)), "prune48_input": int(len(splats.positions))}


if __name__ == "__main__":
    sys.exit(main())

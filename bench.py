"""Benchmark of the sm_100a per-pixel plane-fit path (BASELINE.json metric).

Workload (``config.workload``): BASELINE config 2 at the headline window --
64 frames of 640x480 float32 metres (16-cell Voronoi planes, sigma =
1.425e-3 Z^2, 5% invalid), 5x5 window, both fits (disparity form =
implicit-rgbd, standard = implicit-standard).  A step is one pass of
``fit_pixels`` over the batch; a pixel-fit is one (pixel, formulation) fit, so
a step is 64 * 307200 * 2 pixel-fits.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU; every rank fits its own 64-frame
batch (weak scaling, no collective on the data path); timing is CUDA events
between two barriers, max over ranks.  ``--impl reference`` times the CPU
restatement of the reference's fast path (oracle/, integral backend) on the
host cores instead (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

CONFIG_NAME = "C2"
WINDOW = 5
FRAMES = 64
METRIC = "Mpixel plane-fits/sec (640x480, 5x5 win) and % of HBM roofline"
UNIT = "Mpixel-fits/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
BYTES_IN = 4  # float32 depth
BYTES_OUT = 25  # per pixel per formulation: 12 normal + 4 offset + 4 residual + 4 curvature + 1 status


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def profiled_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("dram_bytes_per_launch", {})
    except Exception:
        return None


def profiled_pipes(kernel: str):
    """What binds the dominant kernel instead of HBM, from the same committed ncu capture:
    issue-slot and pipe utilisation (fractions of peak)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        k = json.loads(p.read_text())["kernels"][kernel]
    except Exception:
        return None

    def pct(name):
        try:
            return float(str(k[name]).split()[0]) / 100.0
        except Exception:
            return None

    return {"bound": "instruction issue under fp64 / MUFU dependency latency",
            "issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe": pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "xu_pipe": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "dram_throughput": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "source": "profiles/ncu_summary.json (ncu --set full)"}


def host_cpu() -> dict:
    """CPU model and the cores this process may run on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "affinity_cores": len(os.sched_getaffinity(0))}


def link_bandwidth(host_out, out, forms, stream) -> float:
    """Device->host bandwidth of one plain pinned copy of a whole step's outputs (GB/s): the
    ceiling the end-to-end pipeline is held to."""
    names = ("normal", "offset", "residual", "curvature", "status")
    pairs = [(getattr(host_out[f], k), getattr(out[f], k)) for f in forms for k in names]
    nbytes = sum(hb.numel() * hb.element_size() for hb, _ in pairs)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for hb, src in pairs:
                hb.copy_(src, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/rf_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2], parts[3], parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return None
        sm = [r[0] for r in rows]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[4]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    from paper_2103_06644_b200.shard import max_over_ranks as _max

    return _max(x, world, "cuda" if torch.cuda.is_available() else "cpu")


# ----------------------------------------------------------------- CPU legs
def cpu_reference_rate(frames_host: torch.Tensor, cfg, budget_s: float, threads: int = 0):
    """Oracle (restated reference fast path: integral backend + Jacobi) on host cores.
    Fits whole frames, both formulations, until budget_s of wall time; returns
    (pixel-fits/s, cores, sample description)."""
    from oracle import oracle as O

    tx, ty = O.tan_maps(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    cores = threads if threads > 0 else O.max_threads()
    fits = 0
    nfr = 0
    t0 = time.perf_counter()
    while True:
        d = frames_host[nfr % frames_host.shape[0]].numpy()
        values, valid = O.depth_from_meters(d)
        for code in (O.RGBD, O.STANDARD):
            O.fit_pixels(values, valid, tx, ty, WINDOW, code, backend=O.INTEGRAL, nthreads=cores)
            fits += d.size
        nfr += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return fits / el, cores, el, (f"{nfr} full 640x480 frame(s) of the workload, both formulations, "
                                  f"integral backend (per-frame SATs + per-pixel box sums + 4x4 Jacobi), "
                                  f"{cores} threads, {el:.1f} s wall")


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2103_06644_b200 import scenes

    cfg = scenes.CONFIGS[CONFIG_NAME]
    frames = scenes.render_batch(cfg, frames=4, device="cpu")
    from oracle import oracle as O

    O.build() if not O.LIB_PATH.exists() else None
    # each step is a bounded sample (whole frames, >= 1) sized so that the whole
    # --steps K --warmup W run stays within about two minutes of wall time
    budget = min(2.0, 100.0 / max(args.steps + args.warmup, 1))
    for _ in range(max(args.warmup, 0)):
        cpu_reference_rate(frames, cfg, 0.0)
    rates = []
    total = 0.0
    for _ in range(args.steps):
        r, cores, el, sample = cpu_reference_rate(frames, cfg, budget)
        rates.append(r)
        total += el
    value = statistics.median(rates) / 1e6
    step_fits = FRAMES * cfg.width * cfg.height * 2
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_fits / (value * 1e6) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Voronoi planes, BASELINE config 2)",
        "config": {"workload": "C2: 64x640x480 f32 depth, window 5, implicit-rgbd + implicit-standard",
                   "note": "each step fits a bounded sample (whole frames for ~2 s); value extrapolates "
                           "pixel-fits/s to the 64-frame step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg
def run_ours(args, world, rank, local):
    import paper_2103_06644_b200 as rf
    from paper_2103_06644_b200 import scenes

    dev = torch.device("cuda", local)
    cfg = scenes.CONFIGS[CONFIG_NAME]
    B, H, W = FRAMES, cfg.height, cfg.width
    from paper_2103_06644_b200.shard import rank_seed_base

    depth = scenes.render_batch(cfg, frames=B, device=dev, seed_base=rank_seed_base(2, rank))
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, W, H)
    maps = rf.compute_tan_maps(cam, dev)
    forms = rf.PIXEL_FORMULATIONS
    out = {f: rf.PixelFits.empty(B, H, W, dev) for f in forms}
    stream = torch.cuda.current_stream(dev)

    def step():
        rf.fit_pixels(depth, maps, WINDOW, forms, out=out, stream=stream)

    # warm-up
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region (value): one fit_pixels call per step fits both
    # formulations (rf.launches_per_call launches: one per space at this batch size)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        e0, e1 = ev[k]
        e0.record(stream)
        rf.fit_pixels(depth, maps, WINDOW, forms, out=out, stream=stream)
        e1.record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    ms_total = start.elapsed_time(end)
    per_call = [e0.elapsed_time(e1) for e0, e1 in ev]
    ms_total = max_over_ranks(ms_total, world)
    ms_step = ms_total / args.steps
    fits_step = B * H * W * len(forms)
    value = world * fits_step / (ms_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel (the fused tile kernel: the whole step)
    peak, peak_src = hbm_peak()
    launches_step = rf.launches_per_call(forms, WINDOW, torch.float32, (B, H, W))
    launch_ms = statistics.mean(per_call) / launches_step
    alg_bytes = B * H * W * (BYTES_IN + BYTES_OUT * len(forms)) // launches_step
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    traffic = None
    tr = profiled_traffic()
    if tr and "fused" in tr:
        traffic = tr["fused"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "fit_tile_kernel<SP, TMA, r=2> (one launch per space)",
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes, "launches_per_step": launches_step,
                "launch_ms": launch_ms, "binding": profiled_pipes("fused")}

    # ---- end to end through the public API with host buffers (pinned): HostPipeline
    host_in = depth.cpu().pin_memory()
    pipe = rf.HostPipeline(maps, WINDOW, forms, chunk_frames=8)
    h2d = host_in.numel() * host_in.element_size()
    host_out = pipe.run(host_in)   # warm-up (allocates the pinned outputs and the device ring)
    d2h = sum(getattr(host_out[f], k).numel() * getattr(host_out[f], k).element_size()
              for f in forms for k in ("normal", "offset", "residual", "curvature", "status"))
    pipe.run(host_in)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pipe.run(host_in)          # returns once the step's outputs are in host memory
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = max_over_ranks(e2e_ms, world)
    e2e_value = world * fits_step * args.steps / (e2e_ms * 1e-3) / 1e6
    link = link_bandwidth(host_out, out, forms, pipe.d2h)

    launches = rf.launches_per_call(forms) * args.steps

    sweep = None
    if rank == 0 and not args.no_sweep:
        del host_in, host_out, pipe
        torch.cuda.empty_cache()
        sweep = config_sweep(dev, peak)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu:
        frames_host = depth[:4].cpu()
        r, cores, el, sample = cpu_reference_rate(frames_host, cfg, args.cpu_seconds)
        r1, _, _, sample1 = cpu_reference_rate(frames_host, cfg, 0.5, threads=1)
        cpu_baseline = {"value": r / 1e6, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                        "value_1core": r1 / 1e6, "sample_1core": sample1, "host": host_cpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 16-cell Voronoi planes, sigma=1.425e-3 Z^2, 5% invalid; BASELINE config 2)",
            "config": {"workload": "C2: 64x640x480 f32 depth per GPU, window 5, implicit-rgbd + implicit-standard",
                       "frames_per_gpu": B, "window": WINDOW, "pixel_fits_per_step_per_gpu": fits_step,
                       "l2": "no flush: 79 MB in + 983 MB out per step > 126 MB L2",
                       "launches_per_step": launches_step,
                       "frames_per_s": world * B / (ms_step * 1e-3)},
            "roofline": roofline,
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "note": "rf.HostPipeline: pinned host in/out, 8-frame chunks, H2D / fit / D2H on three streams",
                    "d2h_gbs_achieved": d2h * args.steps / (e2e_ms * 1e-3) / 1e9,
                    "d2h_gbs_plain_copy": link,
                    "bound": "PCIe device-to-host copy of the outputs (25 B per pixel-fit)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "sweep": sweep,
        }
        print(json.dumps(line), flush=True)


def config_sweep(dev, peak):
    """Informational: steady-state throughput of every BASELINE config shape on this GPU
    (both implicit fits, CUDA events over repeated passes of a representative chunk of
    frames; the bench line above is config 2 at window 5)."""
    import paper_2103_06644_b200 as rf
    from paper_2103_06644_b200 import scenes

    plan = [("C1", 1, (5,)), ("C2", 64, (3, 5, 7, 11, 15)), ("C3", 32, (9,)), ("C4", 16, (15,)), ("C5", 4, (31,))]
    res = {}
    stream = torch.cuda.current_stream(dev)
    for name, frames, windows in plan:
        cfg = scenes.CONFIGS[name]
        depth = scenes.render_batch(cfg, frames=frames, device=dev)
        maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height), dev)
        out = {f: rf.PixelFits.empty(frames, cfg.height, cfg.width, dev) for f in rf.PIXEL_FORMULATIONS}
        for w in windows:
            for _ in range(3):
                rf.fit_pixels(depth, maps, w, out=out, stream=stream)
            reps = 20 if name in ("C1", "C2") else 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                rf.fit_pixels(depth, maps, w, out=out, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            px = frames * cfg.width * cfg.height
            in_b = 2 if cfg.u16 else 4
            res[f"{name}_w{w}"] = {
                "frames": frames, "ms_per_pass": ms, "Mpixel_fits_per_s": 2 * px / (ms * 1e-3) / 1e6,
                "frames_per_s": frames / (ms * 1e-3),
                "hbm_frac": 2 * px * (in_b + BYTES_OUT) / (ms * 1e-3) / 1e9 / peak,
                "full_batch_ms_extrapolated": ms * cfg.frames / frames}
        if name == "C2":
            # all four formulations at the headline window (implicit + explicit share each space's pass)
            out4 = {f: rf.PixelFits.empty(frames, cfg.height, cfg.width, dev) for f in rf.FORMULATIONS}
            for _ in range(3):
                rf.fit_pixels(depth, maps, 5, rf.FORMULATIONS, out=out4, stream=stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(20):
                rf.fit_pixels(depth, maps, 5, rf.FORMULATIONS, out=out4, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            px = frames * cfg.width * cfg.height
            res["C2_w5_all4"] = {"frames": frames, "ms_per_pass": ms,
                                 "Mpixel_fits_per_s": 4 * px / (ms * 1e-3) / 1e6, "formulations": 4}
            del out4
        del depth, out
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the informational per-config sweep")
    args = ap.parse_args()
    if args.impl == "reference":
        # the reference arm is the host-CPU restatement: rank 0 alone runs it, no process group
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), 0)
        return
    world, rank, local = dist_setup()
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

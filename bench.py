"""Benchmark of the sm_100a per-pixel plane-fit path (BASELINE.json metric).

Workload (``config.workload``): BASELINE config 2 at the headline window --
64 frames of 640x480 float32 metres (16-cell Voronoi planes, sigma =
1.425e-3 Z^2, 5% invalid), 5x5 window, both fits (disparity form =
implicit-rgbd, standard = implicit-standard).  A step is one pass of
``fit_pixels`` over the batch; a pixel-fit is one (pixel, formulation) fit, so
a step is 64 * 307200 * 2 pixel-fits per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scaling weak|strong] [--frames F]

N > 1: one rank per GPU over NCCL (the command re-launches itself under
torch.distributed.run when WORLD_SIZE is unset).  weak (default): every rank fits
its own 64-frame batch; strong: one 64-frame batch is split into contiguous frame
ranges (shard.frame_range).  No collective on the data path; timing is CUDA events
between two barriers, max over ranks.  After the timed region the batch is checked
against the oracle (``parity`` in the line; exit 3 on a mismatch).  ``--impl
reference`` times the CPU restatement of the reference's fast path (oracle/,
integral backend) on the host cores instead (rank 0 only).
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
FP64_PEAK_TOPS = 17.1  # measured DFMA throughput, T/s (profiles/peak_probe_r1.txt)
NOMINAL_HBM_GBS = 8000.0  # B200 HBM3e nominal (the roofline itself uses the measured copy bandwidth)


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


def profiled_fp64(kernel: str, launch_ms: float):
    """Secondary roofline: the dominant kernel's executed fp64 instructions per
    launch (committed ncu SASS count) over this run's launch time, against the measured DFMA
    peak (profiles/peak_probe_r1.txt: 17.1 T/s on this pool's B200s)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        n = float(json.loads(p.read_text())["kernels"][kernel]["fp64_thread_inst_per_launch"])
    except Exception:
        return None
    achieved = n / (launch_ms * 1e-3) / 1e12
    return {"achieved": achieved, "peak": FP64_PEAK_TOPS, "unit": "T fp64 inst/s", "frac": achieved / FP64_PEAK_TOPS,
            "fp64_thread_inst_per_launch": n, "peak_source": "measured: tools/peak_probe.cu, profiles/peak_probe_r1.txt"}


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

    return {"bound": "instruction issue under fp64 / MUFU dependency latency (pipes shared in the solve phase)",
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


def dist_setup(stub: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cuda = torch.cuda.is_available() and not stub
    if world > 1:
        import torch.distributed as dist

        if cuda:
            torch.cuda.set_device(local)
        dist.init_process_group(backend="nccl" if cuda else "gloo")
        if rank == 0:
            print(f"bench: process group up, backend {dist.get_backend()}, world {world}", file=sys.stderr, flush=True)
    elif cuda:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    from paper_2103_06644_b200.shard import max_over_ranks as _max
    import torch.distributed as dist

    dev = "cuda" if world > 1 and dist.get_backend() == "nccl" else "cpu"
    return _max(x, world, dev)


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
        # measured wall time per step (a bounded sample of the workload, see config.note)
        "ms_per_step": total / max(args.steps, 1) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Voronoi planes, BASELINE config 2)",
        "config": {"workload": "C2: 64x640x480 f32 depth, window 5, implicit-rgbd + implicit-standard",
                   "note": "each step fits a bounded sample of the workload (whole C2 frames, both "
                           f"formulations, for ~{budget:.2f} s of wall time, at least one frame); value = "
                           "pixel-fits/s of those samples "
                           "(median over steps); a whole 64-frame step would take "
                           f"{step_fits / (value * 1e6):.1f} s at this rate",
                   "sample_seconds_per_step": total / max(args.steps, 1)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg
def shard_plan(args, world: int, rank: int):
    """Frames this rank fits per step and their seeds.  weak: every rank its own FRAMES-frame
    batch (distinct seeds); strong: one FRAMES-frame batch split into contiguous frame ranges
    (shard.frame_range), the seeds of the global frame indices."""
    from paper_2103_06644_b200.shard import frame_range, rank_seed_base

    if args.scaling == "strong":
        start, stop = frame_range(args.frames, world, rank)
        return stop - start, rank_seed_base(2, 0) + start, (start, stop)
    return args.frames, rank_seed_base(2, rank), (0, args.frames)


def parity_check(depth, out, cam, forms, rng_seed: int = 7) -> dict:
    """The timed batch against the oracle (reference naive backend restated in C,
    fitting.py:757-786 and :339-402): every pixel of the shard's first frame, and 2,000 sampled
    pixels (uniform + borders + hole edges) of its last frame, both formulations."""
    import numpy as np

    from oracle.compare import compare
    from tests.helpers import gpu_flat, oracle_frame

    B, H, W = depth.shape
    rng = np.random.default_rng(rng_seed)
    res = {"ok": True, "frames": [0, B - 1], "checks": []}
    last = depth[B - 1].cpu().numpy()
    valid = last > 0
    edge = np.flatnonzero(valid & ~np.roll(valid, 1, axis=1))
    pix = np.unique(np.concatenate([
        rng.choice(H * W, 2000, replace=False),
        np.arange(W), (H - 1) * W + np.arange(W), np.arange(H) * W, np.arange(H) * W + W - 1,
        rng.choice(edge, min(300, edge.size), replace=False) if edge.size else np.zeros(0, np.int64)]))
    for frame, sel in ((0, None), (B - 1, pix)):
        for f in forms:
            ref = oracle_frame(depth[frame].cpu(), cam, WINDOW, f, pixels=sel)
            m = compare(gpu_flat(out[f], frame, sel), ref, explicit_fit=f.startswith("explicit"))
            res["checks"].append({"frame": frame, "form": f, "pixels": m["pixels"], "compared": m["compared"],
                                  "status_mismatch": m["status_mismatch"],
                                  "degenerate_ref": m["degenerate_ref"], "degenerate_mismatch": m["degenerate_mismatch"],
                                  "max_normal_rad": m["max_normal_rad"], "max_residual_rel": m["max_residual_rel"],
                                  "max_curvature_rel": m["max_curvature_rel"], "ok": m["ok"]})
            res["ok"] = res["ok"] and m["ok"]
    res["tolerances"] = {"normal_rad": 1e-4, "residual_rel": 1e-4, "curvature_rel": 1e-4, "status_bits": "exact",
                         "degenerate_bit": "reported (a float threshold, fitting.py:552-554; SURVEY A18)"}
    return res


class _CudaLeg:
    """The measured path: device-resident batch, CUDA events on the launching stream."""

    def __init__(self, local: int):
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream(self.dev)

    def event(self):
        return torch.cuda.Event(enable_timing=True)

    def record(self, ev):
        ev.record(self.stream)

    @staticmethod
    def elapsed(e0, e1) -> float:
        return e0.elapsed_time(e1)

    def sync(self):
        torch.cuda.synchronize(self.dev)


class _StubLeg:
    """CPU stand-in for the control-flow tests (tests/test_bench_multirank.py): host tensors,
    wall-clock 'events', and a torch op in place of the kernel.  Never used for a number."""

    def __init__(self, local: int):
        self.dev = torch.device("cpu")

    def event(self):
        return [0.0]

    def record(self, ev):
        ev[0] = time.perf_counter()

    @staticmethod
    def elapsed(e0, e1) -> float:
        return (e1[0] - e0[0]) * 1e3

    def sync(self):
        pass


def run_ours(args, world, rank, local):
    import paper_2103_06644_b200 as rf
    from paper_2103_06644_b200 import scenes

    stub = args.stub
    leg = _StubLeg(local) if stub else _CudaLeg(local)
    dev = leg.dev
    cfg = scenes.CONFIGS[CONFIG_NAME] if not stub else scenes.small_config(CONFIG_NAME, 64, 48)
    H, W = cfg.height, cfg.width
    B, seed_base, (g0, g1) = shard_plan(args, world, rank)
    depth = scenes.render_batch(cfg, frames=B, device=dev, seed_base=seed_base)
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, W, H)
    forms = rf.PIXEL_FORMULATIONS
    if stub:
        out = None

        def step():
            return (depth * 2.0).sum()
    else:
        maps = rf.compute_tan_maps(cam, dev)
        out = {f: rf.PixelFits.empty(B, H, W, dev) for f in forms}

        def step():
            rf.fit_pixels(depth, maps, WINDOW, forms, out=out, stream=leg.stream)

    for _ in range(max(args.warmup, 3)):
        step()
    leg.sync()

    # ---- device-resident timed region (value): one fit_pixels call per step fits both
    # formulations (rf.launches_per_call launches: one per space at this batch size)
    ev = [[leg.event() for _ in range(2)] for _ in range(args.steps)]
    sampler = None if stub else ClockSampler(local)
    if sampler:
        sampler.start()
        time.sleep(0.3)
    barrier(world)
    leg.sync()
    start, end = leg.event(), leg.event()
    leg.record(start)
    for k in range(args.steps):
        e0, e1 = ev[k]
        leg.record(e0)
        step()
        leg.record(e1)
    leg.record(end)
    leg.sync()
    barrier(world)
    clocks = sampler.stop() if sampler else None
    ms_total = max_over_ranks(leg.elapsed(start, end), world)
    per_call = [leg.elapsed(e0, e1) for e0, e1 in ev]
    ms_step = ms_total / args.steps
    # whole-job pixel-fits per step: the sum over ranks (weak: world x batch; strong: the batch)
    total_frames = args.frames * world if args.scaling == "weak" else args.frames
    fits_step = total_frames * H * W * len(forms)
    value = fits_step / (ms_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel: the tile kernel (one launch per space here)
    peak, peak_src = hbm_peak()
    launches_step = 1 if stub else rf.launches_per_call(forms, WINDOW, torch.float32, (B, H, W))
    launch_ms = statistics.mean(per_call) / launches_step
    # per launch: every launch reads the input once and writes its formulations' outputs
    alg_bytes = B * H * W * (BYTES_IN + BYTES_OUT * len(forms) // launches_step)
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    step_bytes = B * H * W * (BYTES_IN + BYTES_OUT * len(forms))  # the step's compulsory bytes (input once)
    traffic = None
    tr = profiled_traffic()
    if tr and "per_space" in tr:
        traffic = tr["per_space"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "fit_tile_kernel<SP, TMA, r=2> (one launch per space)",
                "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                "algorithmic_bytes_per_pixel_fit": alg_bytes / (B * H * W * len(forms) / launches_step),
                "step_frac": step_bytes / (ms_step * 1e-3) / 1e9 / peak,
                "step_bytes_note": "whole step at 27 B per pixel-fit (input read once for both forms, V=2)",
                "launches_per_step": launches_step, "launch_ms": launch_ms,
                # also against the nominal HBM3e bandwidth (~8 TB/s)
                "nominal": {"peak": NOMINAL_HBM_GBS, "frac": achieved / NOMINAL_HBM_GBS,
                            "step_frac": step_bytes / (ms_step * 1e-3) / 1e9 / NOMINAL_HBM_GBS},
                "fp64": profiled_fp64("per_space", launch_ms),
                "binding": profiled_pipes("per_space")}

    # ---- end to end through the public API with host buffers (pinned): HostPipeline
    e2e = None
    if not stub:
        host_in = depth.cpu().pin_memory()
        pipe = rf.HostPipeline(maps, WINDOW, forms, chunk_frames=8)
        h2d = host_in.numel() * host_in.element_size()
        host_out = pipe.run(host_in)   # warm-up (allocates the pinned outputs and the device ring)
        d2h = sum(getattr(host_out[f], k).numel() * getattr(host_out[f], k).element_size()
                  for f in forms for k in ("normal", "offset", "residual", "curvature", "status"))
        pipe.run(host_in)
        leg.sync()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pipe.run(host_in)          # returns once the step's outputs are in host memory
        leg.sync()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
        e2e_value = fits_step * args.steps / (e2e_ms * 1e-3) / 1e6
        link = link_bandwidth(host_out, out, forms, pipe.d2h)
        e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d * world if args.scaling == "weak" else None,
               "d2h_bytes_per_step": d2h * world if args.scaling == "weak" else None,
               "h2d_bytes_per_step_per_gpu": h2d, "d2h_bytes_per_step_per_gpu": d2h,
               "note": "rf.HostPipeline per rank: pinned host in/out, 8-frame chunks, H2D / fit / D2H on three "
                       "streams; each GPU's own PCIe link",
               "d2h_gbs_achieved_per_gpu": d2h * args.steps / (e2e_ms * 1e-3) / 1e9,
               "d2h_gbs_plain_copy": link,
               "bound": "PCIe device-to-host copy of the outputs (25 B per pixel-fit)"}
        if args.scaling == "strong":
            e2e["h2d_bytes_per_step"] = args.frames * H * W * BYTES_IN
            e2e["d2h_bytes_per_step"] = args.frames * H * W * BYTES_OUT * len(forms)
        del host_in, host_out, pipe

    launches = 0 if stub else rf.launches_per_call(forms, WINDOW, torch.float32, (B, H, W)) * args.steps

    # ---- the timed batch, checked against the oracle (outside the timed region)
    parity = None
    if not stub and not args.no_parity and rank == 0:
        parity = parity_check(depth, out, cam, forms)

    sweep = None
    if rank == 0 and not args.no_sweep and not stub:
        torch.cuda.empty_cache()
        sweep = config_sweep(dev, peak)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu and not stub:
        frames_host = depth[:4].cpu()
        r, cores, el, sample = cpu_reference_rate(frames_host, cfg, args.cpu_seconds)
        r1, _, _, sample1 = cpu_reference_rate(frames_host, cfg, 0.5, threads=1)
        cpu_baseline = {"value": r / 1e6, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                        "value_1core": r1 / 1e6, "sample_1core": sample1, "host": host_cpu()}

    shards = [list(shard_plan(args, world, r)[2]) for r in range(world)]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 16-cell Voronoi planes, sigma=1.425e-3 Z^2, 5% invalid; BASELINE config 2)"
                    + (" [STUB: control-flow test, not a measurement]" if stub else ""),
            "config": {"workload": f"C2: {args.frames}x{H}x{W} f32 depth "
                                   + ("per GPU" if args.scaling == "weak" else "sharded over the GPUs")
                                   + ", window 5, implicit-rgbd + implicit-standard",
                       "frames_per_step": total_frames, "frame_shards": shards, "window": WINDOW,
                       "pixel_fits_per_step": fits_step,
                       "l2": "no flush: 79 MB in + 983 MB out per GPU per step > 126 MB L2",
                       "launches_per_step_per_gpu": launches_step,
                       "frames_per_s": total_frames / (ms_step * 1e-3)},
            "roofline": roofline,
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "parity": parity,
            "gpu_launches": launches,
            "clocks": clocks,
            "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
        if parity is not None and not parity["ok"]:
            print("bench: the timed batch does not match the oracle", file=sys.stderr, flush=True)
            sys.exit(3)


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


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"bench: spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: each GPU fits its own --frames batch; strong: one --frames batch sharded")
    ap.add_argument("--frames", type=int, default=FRAMES)
    ap.add_argument("--cpu-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the informational per-config sweep")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed batch")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)  # CPU control-flow tests only
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world_env == 0:
        sys.exit(spawn_ranks(args))
    if world_env and args.gpus != world_env:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world_env}; measuring {world_env} ranks",
              file=sys.stderr, flush=True)
    if args.impl == "reference":
        # the reference arm is the host-CPU restatement: rank 0 alone runs it, no process group
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            run_reference(args, max(world_env, 1), 0)
        return
    world, rank, local = dist_setup(args.stub)
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""FLR fit+apply benchmark on B200 (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl flr|reference]

A "step" is one pass of the whole hot path -- block moments, moment blur, per-block
solve, blended apply (a5 for --config c4) -- over one
batch of `--frames-per-step` synthetic frames (default 1).  Inputs are resident in
HBM before the timed region; the step rotates through a pool of distinct frames
whose total size exceeds the 126 MB L2 (no cross-step L2 reuse).  The timed region
is K steps replayed from CUDA graphs, bracketed by barrier + synchronize, timed with
CUDA events on the launching stream; the max over ranks is reported.  Per-kernel
durations (for the roofline of the dominant kernel) come from caller-owned CUDA
events the library records between its launches inside the same timed region.

Multi-GPU (one rank per GPU; `--gpus N` outside torchrun re-launches itself under
torch.distributed.run): frames are independent, so every rank denoises its own frames
and NCCL only carries the timing max and checksums after the timed region.  c2 (the
default) gives every rank one frame per step (weak scaling); c5 is the fixed 256-frame
batch split by dist.shard_range (strong scaling) with per-frame checksums gathered in
global frame order (identical for every G: each frame's arithmetic does not depend on
the batch it runs in).

--impl reference times the fp64 CPU oracle (oracle/flr_ref.c) on the host cores on
a bounded sample of the same workload (a band of rows of the frame per step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024

# BASELINE.json configs (SURVEY section 8(d) recipe)
CONFIGS = {
    "c1": dict(workload="C1 64x64 1spp Q=4 (albedo, normal.v, depth, AO), 8x8 blocks", W=64, H=64, Q=4,
               block=8, upsample=1, sigma=10.0),
    "c2": dict(workload="C2 1920x1080 1spp Q=8 (incl. 2 neural guide planes), 8x8 blocks", W=1920, H=1080,
               Q=8, block=8, upsample=1, sigma=10.0),
    "c3": dict(workload="C3 3840x2160 1spp Q=8, sigma=20 (larger window), 8x8 blocks", W=3840, H=2160, Q=8,
               block=8, upsample=1, sigma=20.0),
    "c4": dict(workload="C4 joint denoise+2x upsample: 960x540 1spp radiance, 1920x1080 guides, Q=8",
               W=960, H=540, Q=8, block=4, upsample=2, sigma=10.0),
    "c5": dict(workload="C5 batch of 256 1080p frames (Q=8, 8x8) frame-sharded over GPUs", W=1920, H=1080, Q=8,
               block=8, upsample=1, sigma=10.0, batch=256),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["flr", "reference"], default="flr")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--frames-per-step", type=int, default=None,
                    help="frames per call per GPU (default 1; c5: 32-frame calls over the rank's shard)")
    ap.add_argument("--pool", type=int, default=0, help="distinct frames rotated (0 = auto, > 2x L2)")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every step from Python")
    ap.add_argument("--check", action="store_true", help="parity-check one frame against the oracle")
    ap.add_argument("--no-inputs-ready", action="store_true",
                    help="do not pass FLR_FLAG_INPUTS_READY (every step waits for the previous one first)")
    ap.add_argument("--modulated", action="store_true",
                    help="the paper's albedo protocol (flr_denoise_modulated: demodulate, denoise, remodulate, "
                         "add direct light; SURVEY f1) on the c2 shape")
    ap.add_argument("--guides", choices=["f32", "f16"], default="f32",
                    help="guide plane precision (f16: the fp16 guide network's output, SURVEY f2)")
    return ap.parse_args()


METRIC = "Mpixel/s (FLR fit+apply, 1spp) and ms per frame; % of HBM BW"


# --------------------------------------------------------------------------- helpers
def out_pixels(cfg):
    return cfg["W"] * cfg["upsample"] * cfg["H"] * cfg["upsample"]


def min_bytes_per_frame(cfg):
    """Algorithmic bytes: fp32 input planes read once + output written once."""
    Q, W, H, U, gb = cfg["Q"], cfg["W"], cfg["H"], cfg["upsample"], cfg.get("gbytes", 4)
    lo = W * H
    hi = lo * U * U
    if cfg.get("modulated"):  # guides, radiance, albedo, direct read once; output written once
        return (Q * gb + 4 * 3 * 4) * lo
    if U == 1:
        return (Q * gb + (3 + 3) * 4) * lo
    return (Q * gb + 3 * 4) * lo + Q * gb * hi + 3 * 4 * hi


def _fit_bytes(c):  # Q guide planes + 3 radiance planes read once
    return (c["Q"] * c.get("gbytes", 4) + 3 * 4) * c["W"] * c["H"]


def _apply_bytes(c):  # Q guide planes read + 3 output planes written once
    return (c["Q"] * c.get("gbytes", 4) + 3 * 4) * out_pixels(c)


def _fit_mod_bytes(c):  # + 3 albedo planes
    return _fit_bytes(c) + 3 * 4 * c["W"] * c["H"]


def _apply_mod_bytes(c):  # + 3 albedo and 3 direct-light planes
    return _apply_bytes(c) + 6 * 4 * out_pixels(c)


KERNEL_BYTES = {
    "k_fit_ws_mod": _fit_mod_bytes, "k_apply_ws_mod": _apply_mod_bytes,
    # algorithmic bytes per frame of each launch: the full-resolution planes it must read + write
    "k_fit_moments": _fit_bytes, "k_fit_ws": _fit_bytes, "k_fit_ws_f64acc": _fit_bytes,
    "k_fit_ws_f16": _fit_bytes,
    "k_apply_tile": _apply_bytes, "k_apply_px": _apply_bytes, "k_apply_centered": _apply_bytes,
    "k_apply_ws": _apply_bytes, "k_apply_ws_f16": _apply_bytes,
    "k_flr_wave": lambda c: min_bytes_per_frame(c),
}


def k2_flops_per_frame(c):
    """Algorithmic fp64 flops of K2 per frame: the separable blur (2 passes of 2R+1 taps on
    each of the KM moment components) + the appendix solve (Cholesky Q^3/3, 3 right-hand
    sides 3 Q^2, normalisation and model assembly) per block; FMA = 2 flops."""
    Q, W, H, D = c["Q"], c["W"], c["H"], c["block"]
    R = c.get("radius") or math.ceil(2.0 * c["sigma"] / (D * c["upsample"]) - 1e-12)
    KM = 1 + Q + Q * (Q + 1) // 2 + 3 + 3 * Q
    NS = Q * (Q + 1) // 2
    blocks = -(-W // D) * -(-H // D)
    blur = KM * 2 * (2 * R + 1)
    solve = Q ** 3 / 3 + 3 * Q * Q + 12 * Q + 3 * NS
    return blocks * 2 * (blur + solve)


KERNEL_FLOPS = {  # fp64-bound kernels
    "k_blur_solve_tile": k2_flops_per_frame,
}
# DP peak from the unit count: 148 SMs x 64 FP64 FMA/clk (measured 63/clk/SM with a DFMA
# microbenchmark, tools/ubench_fma.cu) x 2 flops x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel, config):
    """dram__bytes_read+write per launch from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


def step_traffic(config, variant, frames):
    """Whole-step DRAM bytes per call from the committed ncu app-range capture
    (profiles/r02_step_traffic.json, tools/step_traffic.py), c2 single-frame steps only."""
    p = os.path.join(ROOT, "profiles", "r02_step_traffic.json")
    if config != "c2" or frames != 1 or not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))["fused" if variant == 2 else "staged_steady"]
        return {"dram_bytes": d["dram_bytes"], "dram_read_bytes": d["dram_read_bytes"],
                "dram_write_bytes": d["dram_write_bytes"], "bytes_per_output_px": d["dram_bytes_per_output_px"],
                "source": "profiles/r02_step_traffic.json (ncu app-range replay; staged: 8 back-to-back calls "
                          "without cache flushes, per call, incl. write-backs; fused: one call after a flush)"}
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, index, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks_setting": getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sync_boost": getattr(nv, "nvmlClocksEventReasonSyncBoost", 0x10),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg, budget_s, seed=777, one_thread=False):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: bands of
    full-width rows of the frame (multiples of the block size), until ~budget_s."""
    import numpy as np

    import oracle
    from paper_2410_11625_b200 import synth

    W, H, Q, D, U, sigma = cfg["W"], cfg["H"], cfg["Q"], cfg["block"], cfg["upsample"], cfg["sigma"]
    R = math.ceil(2.0 * sigma / (D * U) - 1e-12)
    band = min(H, max(D, (64 // D) * D))
    if U == 1:
        G, Y = synth.frame(W, band, Q=Q, seed=seed)
        G, Y = G.numpy(), Y.numpy()
        run = lambda: oracle.denoise(G, Y, D=D, sigma=sigma, R=R)  # noqa: E731
    else:
        g, y, gh = synth.upsample_pair(W, band, U=U, Q=Q, seed=seed)
        g, y, gh = g.numpy(), y.numpy(), gh.numpy()
        run = lambda: oracle.denoise_upsample(g, y, gh, D_fit=D, U=U, sigma=sigma, R=R)  # noqa: E731
    px = W * band * U * U
    run()  # warm (page-in, thread pool)
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or not times:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    one = None
    if one_thread:  # the same sample on one host thread
        n_thr = oracle.num_threads()
        oracle.set_num_threads(1)
        try:
            t0 = time.perf_counter()
            run()
            t1 = time.perf_counter() - t0
        finally:
            oracle.set_num_threads(n_thr)
        one = {"value": px / t1 / 1e6, "unit": "Mpixel/s", "cores": 1, "sample": f"1 band of {W}x{band} px",
               "ms_per_frame_extrapolated": 1e3 * t1 * (cfg["H"] / band)}
    return {"value": px * len(times) / tot / 1e6, "unit": "Mpixel/s", "cores": oracle.num_threads(),
            "one_thread": one,
            "kind": "oracle", "cpu": cpu_model(),
            "sample": f"{len(times)} bands of {W}x{band} px{' (x%d upsample)' % U if U > 1 else ''} "
                      f"of the {cfg['workload'].split(' ')[0]} workload, {tot:.1f} s",
            "ms_per_frame_extrapolated": 1e3 * tot / len(times) * (cfg["H"] / band)}


# --------------------------------------------------------------------------- reference arm
def ref_config(cfg, R):
    """The config keys both arms print (so the driver can pair the lines)."""
    return {"workload": cfg["workload"], "W": cfg["W"], "H": cfg["H"], "Q": cfg["Q"], "block": cfg["block"],
            "upsample": cfg["upsample"], "sigma": cfg["sigma"], "radius": R, "eps_add": 1e-5, "eps_mul": 1e-4}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    import oracle
    from paper_2410_11625_b200 import synth

    W, H, Q, D, U, sigma = cfg["W"], cfg["H"], cfg["Q"], cfg["block"], cfg["upsample"], cfg["sigma"]
    R = math.ceil(2.0 * sigma / (D * U) - 1e-12)
    # size each step so the whole run takes ~2 minutes at most
    total_steps = args.steps + args.warmup
    cal = oracle_sample(cfg, 1.0)
    px_per_s = cal["value"] * 1e6
    budget_px = 90.0 * px_per_s / max(1, total_steps)
    rows = max(D, int(budget_px / (W * U * U) // D) * D)
    rows = min(rows, H)
    if U == 1:
        G, Y = synth.frame(W, rows, Q=Q, seed=1000)
        G, Y = G.numpy(), Y.numpy()
        step = lambda: oracle.denoise(G, Y, D=D, sigma=sigma, R=R)  # noqa: E731
    else:
        g, y, gh = synth.upsample_pair(W, rows, U=U, Q=Q, seed=1000)
        g, y, gh = g.numpy(), y.numpy(), gh.numpy()
        step = lambda: oracle.denoise_upsample(g, y, gh, D_fit=D, U=U, sigma=sigma, R=R)  # noqa: E731
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    px = W * rows * U * U
    value = px * args.steps / dt / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "Mpixel/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg.get("batch") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scene)",
        "config": ref_config(cfg, R), "sample": f"{W}x{rows} band of the frame per step (fp64 CPU oracle)",
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"{args.steps} steps of a {W}x{rows} band", "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- FLR arm
def batch_plan(batch, rank, world, frames_per_call=32):
    """c5's rank loop plan: rank `rank` of `world` owns frames [lo, hi) of the
    global batch (dist.shard_range), seeded by global frame index; it denoises them in
    `pool` calls of F frames (F = the largest divisor of its shard <= frames_per_call)."""
    from paper_2410_11625_b200 import dist as fd

    lo, hi = fd.shard_range(batch, rank, world)
    nsh = hi - lo
    cap = max(1, min(frames_per_call, nsh))
    F = max(d for d in range(1, cap + 1) if nsh % d == 0)
    return lo, hi, F, nsh // F, [1000 + g for g in range(lo, hi)]


def batch_checksums(call, pool, lo, batch, device=None):
    """Per-frame checksums of the rank's `pool` calls (call(i) returns the [F, 3, H, W]
    output of its i-th call), gathered in global frame order and digested: identical for
    every world size, since each frame's arithmetic does not depend on its batch."""
    import hashlib

    import torch

    from paper_2410_11625_b200 import dist as fd

    rows = torch.cat([fd.per_frame_checksums(call(i)) for i in range(pool)]) if pool else torch.zeros(0, 3)
    full = fd.gather_frame_checksums(rows, lo, batch, device=device)
    return {"frames": batch, "sha256": hashlib.sha256(full.numpy().tobytes()).hexdigest(),
            "all_finite": bool(torch.isfinite(full).all() and (full[:, 2] == 1).all()),
            "frame0": full[0].tolist(), "frame_last": full[-1].tolist(),
            "note": "[sum, max|x|, finite] per frame in global order; identical for every G"}


def run_flr(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import synth

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    W, H, Q, D, U, sigma = cfg["W"], cfg["H"], cfg["Q"], cfg["block"], cfg["upsample"], cfg["sigma"]
    half = args.guides == "f16"
    gbytes = cfg["gbytes"]
    frame_in_bytes = (Q * gbytes + 3 * 4) * W * H + (Q * gbytes * W * H * U * U if U > 1 else 0)
    R = flr.effective_radius(block=D, upsample=U, sigma=sigma)
    from paper_2410_11625_b200 import dist as fd

    batch = cfg.get("batch")
    if batch:  # c5: the fixed global batch, split by frame (strong scaling); a step = one pass over it
        lo, hi, F, pool, seeds = batch_plan(batch, rank, world, args.frames_per_step or 32)
        nsh = hi - lo
        K = args.steps * pool
    else:  # one call per step on `frames_per_step` frames of a rotating pool (> 2x L2)
        lo, hi, nsh = 0, 0, 0
        F = args.frames_per_step or 1
        pool = args.pool or max(2, math.ceil(2.5 * L2_BYTES / (frame_in_bytes * F)))
        seeds = fd.frame_seeds(rank, world, pool * F)  # ranks draw disjoint global frames
        K = args.steps

    # ---- inputs resident in HBM (global frame index -> seed)
    gl, yl, gh, al, dl = [], [], [], [], []
    for i in range(pool):
        if args.modulated:  # the renderer's outputs: modulated radiance, albedo, direct light
            fr = [synth.modulated_frame(W, H, Q=Q, seed=seeds[i * F + j], device=dev) for j in range(F)]
            gl.append(torch.stack([t[0] for t in fr]).contiguous())
            yl.append(torch.stack([t[1] for t in fr]).contiguous())
            al.append(torch.stack([t[2] for t in fr]).contiguous())
            dl.append(torch.stack([t[3] for t in fr]).contiguous())
        elif U == 1:
            g, y = synth.batch(F, W, H, Q=Q, seed0=seeds[i * F], device=dev)
            gl.append(g)
            yl.append(y)
        else:
            trip = [synth.upsample_pair(W, H, U=U, Q=Q, seed=seeds[i * F + j], device=dev) for j in range(F)]
            gl.append(torch.stack([t[0] for t in trip]).contiguous())
            yl.append(torch.stack([t[1] for t in trip]).contiguous())
            gh.append(torch.stack([t[2] for t in trip]).contiguous())
    if half:  # the guide network's fp16 planes: converted once, before the timed region
        gl = [g.to(torch.float16) for g in gl]
        gh = [g.to(torch.float16) for g in gh]
    torch.cuda.synchronize()
    # the timed loop's inputs are resident before the timed region: FLR_FLAG_INPUTS_READY lets
    # each step's moment kernel stream while the previous step's apply drains
    flags = 0 if args.no_inputs_ready else flr.FLAG_INPUTS_READY
    den = flr.Denoiser(F, Q, W, H, device=dev, block=D, upsample=U, sigma=sigma, variant=args.variant, flags=flags)
    outs = [torch.empty_like(den.out) for _ in range(2)]

    def call(i, trace=None):
        k = i % pool
        if args.modulated:
            return den.modulated(gl[k], yl[k], al[k], dl[k], out=outs[i % 2], trace=trace)
        return den(gl[k], yl[k], gh[k] if U > 1 else None, out=outs[i % 2], trace=trace)

    # ---- launch count + optional parity check
    call(0)
    launches_per_step = flr.last_launch_count()
    kernel_names = flr.last_launch_names()
    torch.cuda.synchronize()
    check = None
    if args.check and rank == 0:
        import oracle
        from tests.parity import parity_report

        o = call(0).cpu().numpy()
        g0 = gl[0].float().cpu().numpy()
        y0 = yl[0].cpu().numpy()
        if args.modulated:
            ref = oracle.denoise_modulated(g0, y0, al[0].cpu().numpy(), dl[0].cpu().numpy(), D=D, sigma=sigma, R=R)
        elif U == 1:
            ref = oracle.denoise(g0, y0, D=D, sigma=sigma, R=R)
        else:
            ref = oracle.denoise_upsample(g0, y0, gh[0].float().cpu().numpy(), D_fit=D, U=U, sigma=sigma, R=R)
        check = parity_report(o, ref)

    stream = torch.cuda.current_stream(dev)
    n_ev = launches_per_step + 1

    def make_events(n):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for e in evs:
            e.record(stream)
        return evs

    # per-step traces for one pool rotation (reused every replay)
    traces = [flr.EventTrace.from_events(make_events(n_ev)) for _ in range(pool)]

    # ---- warm-up (untimed)
    for i in range(max(3, args.warmup)):
        call(i)
    torch.cuda.synchronize()

    # ---- CUDA graphs: whole pool rotations and the remainder (timed), a traced rotation
    use_graph = not args.no_graph
    G_STEPS = pool * max(1, -(-32 // pool))  # steps per timed graph
    graphs = {}
    if use_graph:
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for i in range(pool):  # warm allocations on the capture stream
                call(i)
        torch.cuda.synchronize()

        def capture(nsteps, traced):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for i in range(nsteps):
                    call(i, trace=traces[i] if traced else None)
            return g

        # the timed graphs carry no events between kernels (an event node would serialise
        # the programmatic-dependent launches); per-kernel durations come from a traced
        # replay of the same steps right after the timed region.  A timed graph holds several
        # pool rotations (>= 32 steps): the programmatic-dependent chain -- each step's moment
        # kernel streaming while the previous apply drains -- breaks at every graph launch, as
        # it would not in a renderer's continuous frame loop
        reps, rem = divmod(K, G_STEPS)
        if reps:
            graphs["full"] = capture(G_STEPS, False)
        if rem:
            graphs["rem"] = capture(rem, False)
        graphs["traced"] = capture(pool, True)
        torch.cuda.synchronize()

    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank if "CUDA_VISIBLE_DEVICES" not in os.environ else local_rank)
    with sampler:
        time.sleep(0.02)
        t_start.record(stream)
        if use_graph:
            reps, rem = divmod(K, G_STEPS)
            for _ in range(reps):
                graphs["full"].replay()
            if rem:
                graphs["rem"].replay()
        else:
            for i in range(K):
                call(i)
        t_stop.record(stream)
        torch.cuda.synchronize()
        # traced pass (not part of the value): events between the kernels of each step
        per_kernel_acc = {n: [] for n in kernel_names}
        for _ in range(max(1, min(K, 400) // pool)):
            if use_graph:
                graphs["traced"].replay()
            else:
                for i in range(pool):
                    call(i, trace=traces[i])
            torch.cuda.synchronize()
            for tr in traces:
                evs = tr._keep[1]
                for j in range(min(len(kernel_names), tr.recorded - 1 if tr.recorded else len(evs) - 1)):
                    per_kernel_acc[kernel_names[j]].append(evs[j].elapsed_time(evs[j + 1]))
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_stop)
    clocks = sampler.summary()

    # per-launch durations from the traced pass (launch gaps included)
    names = kernel_names
    per_kernel = per_kernel_acc
    avg_ms = {n: (sum(v) / len(v) if v else None) for n, v in per_kernel.items()}

    ms_max = fd.max_over_ranks(ms, device=dev)

    # ---- end-to-end through the C ABI with host buffers (pinned), copies inside the timed region
    E = max(1, args.e2e_steps)
    e2e = None
    if E:
        # End to end through the C ABI from pinned host buffers, the way a renderer streams
        # frames: step i's host->device copy, its denoise call and its device->host copy run on
        # three streams with double-buffered device inputs/outputs, so frame i+1 uploads while
        # frame i computes and frame i-1 downloads; every byte of every step moves inside the
        # timed region.
        hp = min(pool, 2)
        pin = lambda lst: [lst[k].cpu().pin_memory() for k in range(hp)] if lst else None  # noqa: E731
        h_in = {"g": pin(gl), "y": pin(yl), "gh": pin(gh) if U > 1 else None,
                "a": pin(al) if args.modulated else None, "dl": pin(dl) if args.modulated else None}
        h_out = [den.out.cpu().pin_memory() for _ in range(2)]
        d_in = [{k: (torch.empty_like(v[0].to(dev)) if v else None) for k, v in h_in.items()} for _ in range(2)]
        d_out = [torch.empty_like(den.out) for _ in range(2)]
        h2d = sum(v[0].numel() * v[0].element_size() for v in h_in.values() if v)
        d2h = h_out[0].numel() * 4
        s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("up", "comp", "down")}
        for k in ev:
            for e in ev[k]:
                e.record(stream)

        def e2e_step(i):
            b = i % 2
            k = i % hp
            with torch.cuda.stream(s_up):
                s_up.wait_event(ev["comp"][b])  # inputs of step i-2 consumed
                for name, hv in h_in.items():
                    if hv:
                        d_in[b][name].copy_(hv[k], non_blocking=True)
                ev["up"][b].record(s_up)
            stream.wait_event(ev["up"][b])
            stream.wait_event(ev["down"][b])  # output buffer of step i-2 downloaded
            di = d_in[b]
            if args.modulated:
                den.modulated(di["g"], di["y"], di["a"], di["dl"], out=d_out[b])
            else:
                den(di["g"], di["y"], di["gh"], out=d_out[b])
            ev["comp"][b].record(stream)
            with torch.cuda.stream(s_down):
                s_down.wait_event(ev["comp"][b])
                h_out[b].copy_(d_out[b], non_blocking=True)
                ev["down"][b].record(s_down)

        for i in range(4):
            e2e_step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s_up.wait_event(a)
        s_down.wait_event(a)
        for i in range(E):
            e2e_step(i)
        stream.wait_stream(s_up)
        stream.wait_stream(s_down)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = fd.max_over_ranks(a.elapsed_time(b), device=dev)
        e2e = {"value": world * E * F * out_pixels(cfg) / (e_ms * 1e-3) / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / E, "steps": E,
               "pipeline": "h2d / denoise / d2h on 3 streams, double-buffered (pinned host memory)"}

    # ---- per-frame checksums gathered over NCCL in global frame order (the only collective)
    frame_cs = batch_checksums(call, pool, lo, batch, device=dev) if batch else None
    o = call(0)
    torch.cuda.synchronize()
    allcs = fd.gather_rows(fd.output_checksum(o), device=dev)

    if rank != 0:
        return
    peak, peak_src = load_peaks()
    frames_total = args.steps * batch if batch else world * K * F
    px_total = frames_total * out_pixels(cfg)
    value = px_total / (ms_max * 1e-3) / 1e6
    # dominant kernel (largest share of the step) and its own algorithmic bytes
    known = {n: t for n, t in avg_ms.items() if t}
    # frames one launch of a kernel processes: batched calls whose frames fit in L2 run frame by
    # frame (one fit / K2 / apply launch per frame), the others one launch per call
    fpl = {n: F / max(1, kernel_names.count(n)) for n in known}
    # dominant kernel: the largest share of the step (launch time x launches per call)
    dom = max(known, key=lambda n: known[n] * kernel_names.count(n)) if known else None
    roof = None
    if dom:
        bytes_fn = KERNEL_BYTES.get(dom)
        alg = bytes_fn(cfg) * fpl[dom] if bytes_fn else None
        if alg is not None:
            ach = alg / (known[dom] * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": ncu_traffic(dom, args.config),
                    "algorithmic_bytes_per_launch": alg, "avg_launch_us": known[dom] * 1e3,
                    "peak_source": peak_src}
        elif dom in KERNEL_FLOPS:
            ach = KERNEL_FLOPS[dom](cfg) * fpl[dom] / (known[dom] * 1e-3) / 1e12
            roof = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                    "unit": "TFLOP/s (fp64)", "frac": ach / FP64_PEAK_TFLOPS, "traffic": ncu_traffic(dom, args.config),
                    "avg_launch_us": known[dom] * 1e3, "peak_source": "derived: 148 SM x 64 DFMA/clk x 1.965 GHz"}
        else:
            roof = {"bound": "alu", "kernel": dom, "achieved": None, "peak": None, "unit": None, "frac": None,
                    "traffic": None, "avg_launch_us": known[dom] * 1e3}
    # every kernel against its own roof (bytes for the streaming kernels, fp64 flops for K2)
    kroof = {}
    for n, t in known.items():
        if n in KERNEL_BYTES:
            a_ = KERNEL_BYTES[n](cfg) * fpl[n] / (t * 1e-3) / 1e9
            kroof[n] = {"bound": "hbm", "achieved": a_, "peak": peak, "unit": "GB/s", "frac": a_ / peak,
                        "avg_launch_us": t * 1e3}
        elif n in KERNEL_FLOPS:
            a_ = KERNEL_FLOPS[n](cfg) * fpl[n] / (t * 1e-3) / 1e12
            kroof[n] = {"bound": "alu", "achieved": a_, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s (fp64)",
                        "frac": a_ / FP64_PEAK_TFLOPS, "avg_launch_us": t * 1e3}
    step_ms = ms_max / args.steps  # c5: one pass over the rank's shard of the batch
    step_bytes = min_bytes_per_frame(cfg) * (nsh if batch else F)
    step_roof = {"min_bytes_per_step": step_bytes, "achieved": step_bytes / (step_ms * 1e-3) / 1e9,
                 "peak": peak, "unit": "GB/s", "frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak,
                 "traffic": step_traffic(args.config, args.variant, F)}
    cpu_base = None
    if world == 1 and not args.no_cpu_baseline:
        cpu_base = oracle_sample(cfg, args.cpu_seconds, one_thread=True)
    frames_per_step = batch if batch else world * F
    line = {
        "metric": METRIC,
        "value": value, "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "ms_per_frame": ms_max / frames_total, "frames_per_s": frames_total / (ms_max * 1e-3),
        "higher_is_better": True, "scaling": "strong" if batch else "weak", "vs_baseline": None,
        "dtype": "f32" if not half else "f32 (fp16 guide planes)", "data": "synthetic (seeded procedural Lambertian scenes, rasterised guides, 1spp noise)",
        "config": {**ref_config(cfg, R), "frames_per_call": F, "calls_per_step": pool if batch else 1,
                   "global_batch": frames_per_step, "shard": [lo, hi] if batch else None,
                   "pool_frames": pool * F, "l2": f"inputs rotate through {pool * F} distinct resident frames "
                   f"({pool * F * frame_in_bytes / 1e6:.0f} MB > 126 MB L2)", "graphs": use_graph, "steps_per_graph": (G_STEPS if use_graph else None),
                   "parallelism": f"frame-sharded dp{world}", "variant": args.variant,
                   "guides": args.guides, "modulated": bool(args.modulated),
                   "flags": "FLR_FLAG_INPUTS_READY" if not args.no_inputs_ready else "0",
                   "numerics": "fp32 streams, fp64 block blur+solve"
                               + ("; fp16 guide planes widened exactly to fp32 on load" if half else "")},
        "roofline": roof, "step_roofline": step_roof,
        "kernel_us": {n: (t * 1e3 if t else None) for n, t in avg_ms.items()},
        "kernel_roofline": kroof,
        "cpu_baseline": cpu_base, "e2e": e2e, "gpu_launches": launches_per_step * K,
        "clocks": clocks,
        "checksums": allcs, "frame_checksums": frame_cs,
        "paper_context": {"rtx2080ti_ms_per_1080p_frame": 0.636, "source": "P:429 (Table 1)"},
    }
    if check is not None:
        line["parity"] = check
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    cfg["gbytes"] = 2 if args.guides == "f16" else 4
    if args.modulated:
        if args.config != "c2" or args.guides != "f32":
            sys.exit("--modulated runs on the c2 shape with fp32 guides")
        cfg["modulated"] = True
        cfg["workload"] = "C2 albedo protocol: demodulate, 1080p Q=8 FLR, remodulate + direct light (SURVEY f1)"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    if world != args.gpus:
        sys.exit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_flr(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()

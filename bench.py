#!/usr/bin/env python
"""bench.py -- throughput of the fast adaptive bilateral filter on B200.

Workload (BASELINE.json metric / configs[3]): one 3840x2160 grey frame, box
window rho=20 (41x41), N=8, sigma ~ U[5,60], theta = f + U[-15,15] (synthetic
Voronoi-256 + noise sd 20 stand-in for the paper's photographs).
A "step" is one full pass of the hot path (bounds, moments, fit, integrals,
ratio, exact-moment fallback) over one frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun: every rank filters its own frame (independent
problems, no data-path collective), timing is the max over ranks (weak
scaling).  ``--impl reference`` times the CPU oracle (oracle/, __float128
Algorithm 1) on a bounded pixel sample of the same workload on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpix/s of fast adaptive bilateral filter (4K, rho=20, N=8)"
CFG = 4


def _load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.path = None

    def __enter__(self):
        import tempfile

        try:
            fd, self.path = tempfile.mkstemp(prefix="fabf_clocks_", suffix=".csv")
            self.fh = os.fdopen(fd, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()
            try:
                with open(self.path) as f:
                    self.lines = [ln.strip() for ln in f]
                os.unlink(self.path)
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# B200 FP64 pipe: 64 FMA/clk/SM (microbench: 1.71e13 FMA/s at the clocks seen,
# profiles/r1_microbench.json) x 148 SMs x 1.965 GHz max clock x 2 flop/FMA.
FP64_PEAK_TFLOPS = 64 * 148 * 1.965e9 * 2 / 1e12  # 37.2, derived from unit counts and clocks
FP64_MICROBENCH_TFLOPS = 34.19  # tools/microbench.cu, profiles/r1_microbench.json
FP64_PEAK_SOURCE = ("derived from unit counts and clocks: 64 FP64 FMA/clk/SM x 148 SMs x 1.965 GHz x 2 "
                    "= 37.2 TF/s (not driver-measured; tools/microbench.cu measured 34.2 TF/s)")
J_STAGE_FP64 = 200  # fp64 J-stage (seeds + recurrence) of a lambda >= 2 pixel, ~170-230


def alg_fp64_flops_per_pixel(N: int, share_fp64_j: float, share_identity: float = 0.0) -> float:
    """ALGORITHMIC fp64 flops per pixel: moments 6N, stretch +
    Legendre 1.5N^2 + 3.5N, and the fp64 J-stage (~200) only for the share of
    pixels that need it (lambda >= 2 or theta far outside [alpha, beta]; the
    lambda < 2 pixels use fp32 quadrature, no fp64); identity pixels (alpha ==
    beta) do no per-pixel work.  The share comes from one diagnostic call
    outside the timed region (regime codes, fabf_filter_diag)."""
    per = 6 * N + 1.5 * N * N + 3.5 * N
    return (1.0 - share_identity) * per + share_fp64_j * J_STAGE_FP64


def _ncu_summary(kernel: str):
    """Executed-pipe figures of ``kernel`` from the committed ncu --set full
    capture summary (profiles/traffic.json, written by tools/ncu_traffic.py), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f).get(kernel, {})
        return dict(d, source=d.get("report"))
    except Exception:
        return {}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def regime_mix(fb, plan, img, th, sg, rho, N):
    """Shares of identity, small-lambda (fp32 J) and fp64-J pixels, from the
    per-pixel codes of one fabf_filter_diag call (outside any timed region)."""
    import torch

    _, d = fb.filter_diag(plan, img, th, sg, rho, N)
    code = d["code"]
    n = code.numel()
    ident = int(((code & fb.CODE_IDENTITY) > 0).sum())
    small = int(((code & fb.CODE_SMALL_LAMBDA) > 0).sum())
    torch.cuda.synchronize()
    return {"identity": ident / n, "small_lambda_fp32": small / n,
            "fp64_j": (n - ident - small) / n}


def _traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel`` from
    the committed ncu --set full capture summary (tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d[kernel]["dram_bytes"]
    except Exception:
        return None


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_sample(w, npx: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(w.img.size, npx, replace=False))


def time_oracle(w, npx: int, threads: int | None = None, seed: int = 0):
    import oracle

    oracle.build()
    idx = cpu_sample(w, npx, seed)
    t = time.perf_counter()
    oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N, pixels=idx, threads=threads)
    dt = time.perf_counter() - t
    return npx / dt / 1e6, dt


def oracle_sample_size(w, seconds: float) -> int:
    """Pixels of a seeded sample the oracle finishes in about ``seconds`` on
    this host (calibrated on a 2000-pixel sample)."""
    rate, _ = time_oracle(w, 2000, seed=1)
    return int(max(2000, min(w.img.size, rate * 1e6 * seconds)))


def run_reference(args):
    """--impl reference: the oracle as it stands on this host's cores."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import workloads

    w = workloads.config(CFG)
    cores = os.cpu_count() or 1
    # each step is a bounded sample sized so the whole run takes a few minutes
    per_step = max(5.0, min(30.0, args.ref_seconds * 10 / max(1, args.steps + args.warmup)))
    npx = args.ref_pixels or oracle_sample_size(w, per_step)
    for i in range(args.warmup):
        time_oracle(w, max(64, npx // 10), seed=100 + i)
    times = []
    for i in range(args.steps):
        _, dt = time_oracle(w, npx, seed=i)
        times.append(dt)
    tot = sum(times)
    value = args.steps * npx / tot / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpix/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f128", "data": "synthetic",
        "config": {"workload": w.name, "sample": f"{npx} seeded pixels per step of the 8.29 Mpx frame"},
        "roofline": None,
        "cpu_baseline": {"value": value, "unit": "Mpix/s", "cores": cores, "kind": "oracle",
                         "sample": f"{npx} seeded pixels of {w.name} per step"},
        "e2e": {"value": value, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1811_02308_b200 as fb
    from paper_1811_02308_b200 import build

    build.build()
    import workloads
    from paper_1811_02308_b200.shard import frame_shard

    # N > 1: a batch of one config-4 frame per GPU, sharded over the ranks
    # (frame_shard: rank r owns frame r; frame 0 is the BASELINE frame, the
    # others are drawn from the same recipe with their own seeds) -- no
    # data-path collective, each rank filters and keeps its own frame
    first, count = frame_shard(ws, ws, rank)
    assert count == 1
    w = workloads.config(CFG, frame=first)
    B, H, W = w.shape
    px = B * H * W
    img = torch.from_numpy(w.img).to(dev)
    th = torch.from_numpy(w.theta).to(dev)
    sg = torch.from_numpy(w.sigma).to(dev)
    out = torch.empty_like(img)
    plan = fb.Plan(B, H, W)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    clk = ClockSampler(local).__enter__()
    # clock ramp: ~0.2 s of L2-flush writes (no filter work) so that the SM
    # clocks are up before the W warm-up steps (which alone last ~1.5 ms)
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 0.2:
        for _ in range(20):
            flush.fill_(0.0)
        torch.cuda.synchronize()
    wev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for e in wev:
        e.record(stream)  # torch creates the event handle lazily, at first record
    for i in range(max(3, args.warmup)):  # the timed loop's own calls, untimed
        flush.fill_(float(i))
        fb.filter_events(plan, img, th, sg, w.rho, w.N, wev, out=out)
    torch.cuda.synchronize()
    launches_per_step = plan.last_launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    # five CUDA events per step around the step's kernels (fabf_filter_events,
    # recorded on the launch stream, no host sync inside the timed region)
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for evs in kev:
        for e in evs:
            e.record(stream)  # creates the handles before the timed region
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # timed region 1 (the headline): the user's call, fabf_filter, nothing
    # between its kernels (they chain by programmatic dependent launch)
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (outside the events)
        starts[i].record(stream)
        fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
        ends[i].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # timed region 2: the same K steps through fabf_filter_events -- five CUDA
    # events on the launch stream around the step's kernels give each kernel's
    # duration (the events between the kernels cost the PDL overlap, so this
    # region's step time is reported separately, not as the headline)
    istarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    iends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(float(i))
        istarts[i].record(stream)
        fb.filter_events(plan, img, th, sg, w.rho, w.N, kev[i], out=out)
        iends[i].record(stream)
    torch.cuda.synchronize()
    istep_ms = [s.elapsed_time(e) for s, e in zip(istarts, iends)]
    stage = np.zeros(4)
    for evs in kev:
        stage += np.array([evs[j].elapsed_time(evs[j + 1]) for j in range(4)])
    stage /= args.steps
    tot_ms = float(sum(step_ms))
    fallback = plan.last_fallback_count()
    clk.__exit__(None, None, None)
    mix = regime_mix(fb, plan, img, th, sg, w.rho, w.N)  # outside the timed region
    fused = {} if args.no_other_configs else fused_variant(fb, w, img, th, sg, flush)
    colour = {} if args.no_other_configs else colour_variant(fb, dev, flush)
    sharpen = {} if args.no_other_configs else sharpen_variant(fb, dev, flush)
    texture = {} if args.no_other_configs else texture_variant(fb, dev, flush)
    gauss = {} if args.no_other_configs else gauss_variant(fb, dev, flush)
    others = {} if args.no_other_configs else other_configs(fb, dev, flush)

    # end to end through the C ABI with host buffers (pinned), copies inside
    e2e_steps, e2e_s = 0, 0.0
    if not args.no_e2e:
        h_img = torch.from_numpy(w.img).pin_memory()
        h_th = torch.from_numpy(w.theta).pin_memory()
        h_sg = torch.from_numpy(w.sigma).pin_memory()
        h_out = torch.empty_like(h_img).pin_memory()
        fb.filter_host(plan, h_img, h_th, h_sg, w.rho, w.N, h_out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(3, min(args.steps, 20))
        for _ in range(e2e_steps):
            fb.filter_host(plan, h_img, h_th, h_sg, w.rho, w.N, h_out)
        e2e_s = time.perf_counter() - t0

    from paper_1811_02308_b200.shard import max_over_ranks, whole_job_rate

    tot_ms = max_over_ranks(tot_ms, dev)  # device time, max over ranks
    e2e_s = max_over_ranks(e2e_s, dev)
    value = whole_job_rate(px, args.steps, tot_ms * 1e-3, ws)
    e2e_value = whole_job_rate(px, e2e_steps, e2e_s, ws) if e2e_steps else None

    if rank == 0:
        peaks, peak_src = _load_peaks()
        ms = tot_ms / args.steps
        alg_bytes = 16.0 * px  # f, theta, sigma read + g written, fp32
        hbm = {"bound": "hbm", "achieved": alg_bytes / (ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
               "unit": "GB/s", "frac": alg_bytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
               "traffic": None, "peak_source": peak_src, "scope": "whole step, 16 B/px"}
        kf_ms = float(stage[2])  # dominant kernel k_filter, CUDA events on the launch stream
        fpp = alg_fp64_flops_per_pixel(w.N, mix["fp64_j"], mix["identity"])
        flops = fpp * px
        ach = flops / (kf_ms * 1e-3) / 1e12
        nc = _ncu_summary("k_filter")
        fp64 = {"bound": "alu", "pipe": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP64_PEAK_TFLOPS, "traffic": _traffic("k_filter"), "kernel": "k_filter",
                "kernel_ms": kf_ms, "kernel_share_of_step": kf_ms / float(np.median(istep_ms)),
                "alg_flops_per_pixel": fpp,
                "alg_flops_recipe": "SURVEY.md 8(d): 6N moments + 1.5N^2+3.5N stretch + 200 fp64 J-stage "
                                    "on the fp64-J share of pixels",
                "regime_mix": mix,
                "peak_source": FP64_PEAK_SOURCE,
                "frac_of_microbench_peak": ach / FP64_MICROBENCH_TFLOPS,
                "executed_fp64_pipe_util_ncu": nc.get("fp64_pipe_pct"),
                "issue_active_ncu": nc.get("issue_active_pct"),
                "ncu_source": nc.get("source")}
        line = {
            "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": w.name, "height": H, "width": W, "rho": w.rho, "N": w.N,
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "parallelism": f"{ws} frames sharded one per GPU (frame_shard), no data-path collective"
                       if ws > 1 else "1 GPU"},
            "roofline": fp64,
            "hbm_roofline": hbm,
            "step_ms": {"min": min(step_ms), "median": float(np.median(step_ms)), "max": max(step_ms),
                        "argmax": int(np.argmax(step_ms))},
            "fallback_pixels": fallback,
            "stage_ms": {"k_bounds": stage[0] + stage[1], "k_filter": stage[2], "k_fallback": stage[3],
                         "source": "timed region 2: fabf_filter_events, CUDA events between the kernels",
                         "instrumented_step_ms_median": float(np.median(istep_ms))},
            "e2e": {"value": e2e_value, "unit": "Mpix/s", "h2d_bytes_per_step": 12 * px,
                    "d2h_bytes_per_step": 4 * px,
                    "path": "fabf_filter_host: pinned host buffers, row-band pipelined H2D / kernels / D2H"},
            "gpu_launches": launches_per_step * args.steps,  # fabf_last_launch_count x steps
            "launches_per_step": launches_per_step,
            "other_configs": others,
            "fused_variant": fused,
            "colour_variant": colour,
            "sharpen_variant": sharpen,
            "texture_variant": texture,
            "gauss_variant": gauss,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            npx = args.ref_pixels or oracle_sample_size(w, args.ref_seconds)
            v, dt = time_oracle(w, npx)
            line["cpu_baseline"] = {"value": v, "unit": "Mpix/s", "cores": cores, "kind": "oracle",
                                    "cpu_model": _cpu_model(),
                                    "sample": f"{npx} seeded pixels of {w.name} ({dt:.1f} s, "
                                              "__float128 Algorithm 1, all host threads)"}
        line["paper_context"] = PAPER_CONTEXT
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


PAPER_CONTEXT = ("context only, not a target: the paper's MATLAB 9.1 implementation on a 3.4 GHz CPU "
                 "(P:540) takes 171-189 ms for a 512x512 image at N=5 (1.4-1.5 Mpix/s) against 3.9-12.4 s "
                 "for brute force (Table II, P:574-577): 'at least 20x' (P:90, P:564)")


def other_configs(fb, dev, flush, steps: int = 10):
    """Device-timed Mpix/s of BASELINE configs 1-3 (full size, L2 flushed
    between steps, CUDA events) -- reported beside the headline config."""
    import torch

    import workloads

    res = {}
    stream = torch.cuda.current_stream()
    for cfg in (1, 2, 3):
        w = workloads.config(cfg)
        img, th, sg = (torch.from_numpy(a).to(dev) for a in (w.img, w.theta, w.sigma))
        out = torch.empty_like(img)
        plan = fb.Plan(*w.shape)
        for _ in range(3):
            fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.fill_(1.0)
            a.record(stream)
            fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
            b.record(stream)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        res[w.name] = {"Mpix/s": w.img.size / (ms * 1e-3) / 1e6, "ms": ms, "rho": w.rho, "N": w.N,
                       "launches": plan.last_launch_count()}
    return res


def fused_variant(fb, w, img, th, sg, flush, steps: int = 10):
    """The same workload with FABF_FLAG_FUSED (bounds inside k_filter: one pass
    reading f, theta, sigma, writing g-hat -- SURVEY a9), device-timed the same
    way; reported beside the default (bounds kernel + k_filter at rho > 5)."""
    import torch

    plan = fb.Plan(*w.shape, fb.FLAG_FUSED)
    out = torch.empty_like(img)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.fill_(1.0)
        a.record(stream)
        fb.filter(plan, img, th, sg, w.rho, w.N, out=out)
        b.record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    return {"Mpix/s": w.img.size / (ms * 1e-3) / 1e6, "ms_per_step": ms, "launches": plan.last_launch_count(),
            "flags": "FABF_FLAG_FUSED"}


def colour_variant(fb, dev, flush, steps: int = 10):
    """NEXT-3: a 3840x2160 RGB frame (channel-interleaved fp32; the channels are
    the config-4 image, a shifted copy and its negative), rho = 20, N = 8, through
    fabf_filter_interleaved (channel by channel); device-timed,
    colour pixels (3 channels) per second."""
    import torch

    import workloads

    rng = np.random.default_rng(4242)
    base = workloads.config(4).img[0]
    img = np.stack([base, np.roll(base, 97, axis=1), 255 - base], axis=-1)
    th = (img + rng.uniform(-15, 15, img.shape)).astype(np.float32)
    sg = rng.uniform(5, 60, img.shape).astype(np.float32)
    H, W, C = img.shape
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
    img_d, th_d, sg_d = t(img), t(th), t(sg)
    out = torch.empty_like(img_d)
    plan = fb.Plan(C, H, W)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        fb.filter_interleaved(plan, img_d, th_d, sg_d, 20, 8, out=out)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.fill_(1.0)
        a.record(stream)
        fb.filter_interleaved(plan, img_d, th_d, sg_d, 20, 8, out=out)
        b.record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    return {"workload": "3840x2160x3 interleaved RGB, rho=20, N=8", "colour Mpix/s": H * W / (ms * 1e-3) / 1e6,
            "plane Mpix/s": C * H * W / (ms * 1e-3) / 1e6, "ms_per_frame": ms, "launches": plan.last_launch_count()}


def sharpen_variant(fb, dev, flush, steps: int = 10):
    """NEXT-2: the sharpening application at the paper's Fig.4 size
    (1024x1024, rho = 5, N = 5; synthetic Voronoi + noise stand-in) and at 4K
    (rho = 20, N = 8): theta, sigma produced on the device from f alone
    (fabf_filter_sharpen).  Device-timed Mpix/s, and end to end with the
    pinned-host image uploaded and the result read back every frame (4 + 4
    bytes per pixel instead of 12 + 4)."""
    import torch

    import workloads

    res = {}
    for name, (H, W, rho, N) in {"sharpen_1024_rho5_N5": (1024, 1024, 5, 5),
                                 "sharpen_4k_rho20_N8": (2160, 3840, 20, 8)}.items():
        f = workloads.voronoi(H, W, seed=7000 + H, n_seeds=128, noise_sd=12.0).astype(np.float32)[None]
        img = torch.from_numpy(f).to(dev)
        out = torch.empty_like(img)
        plan = fb.Plan(1, H, W)
        stream = torch.cuda.current_stream()
        for _ in range(3):
            fb.filter_sharpen(plan, img, rho, N, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.fill_(1.0)
            a.record(stream)
            fb.filter_sharpen(plan, img, rho, N, out=out)
            b.record(stream)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        h_img = torch.from_numpy(f).pin_memory()
        h_out = torch.empty_like(h_img).pin_memory()
        t0 = time.perf_counter()
        for _ in range(steps):
            img.copy_(h_img, non_blocking=True)
            fb.filter_sharpen(plan, img, rho, N, out=out)
            h_out.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_s = (time.perf_counter() - t0) / steps
        res[name] = {"Mpix/s": H * W / (ms * 1e-3) / 1e6, "ms": ms, "launches": plan.last_launch_count(),
                     "e2e Mpix/s": H * W / e2e_s / 1e6, "e2e_ms": e2e_s * 1e3,
                     "h2d_bytes_per_frame": 4 * H * W, "d2h_bytes_per_frame": 4 * H * W,
                     "params": dict(fb.SHARPEN_DEFAULTS)}
    return res


def texture_variant(fb, dev, flush, steps: int = 10):
    """NEXT-2: the texture-filtering application (fabf_filter_texture):
    the mRTV sigma map on the device, two smoothing passes and the sharpening
    pass (Algorithm 1 three times) from f alone.  Three 650x500 planes of the
    synthetic texture generator (the paper's Fig.11 images are about 500x650
    colour, filtered channel by channel, 2.5 s in its MATLAB implementation; here
    every plane gets its own map) at rho = 5, N = 5, and a 4K plane at rho = 10,
    N = 5.  Device-timed Mpix/s of output pixels, and end to end (image up,
    result down: 4 + 4 bytes per pixel)."""
    import torch

    import workloads

    res = {}
    for name, (B, H, W, rho, N) in {"texture_3x650x500_rho5_N5": (3, 650, 500, 5, 5),
                                    "texture_4k_rho10_N5": (1, 2160, 3840, 10, 5)}.items():
        f = np.stack([workloads.texture(H, W, seed=7700 + 10 * b + B) for b in range(B)]).astype(np.float32)
        img = torch.from_numpy(f).to(dev)
        out = torch.empty_like(img)
        plan = fb.Plan(B, H, W)
        stream = torch.cuda.current_stream()
        for _ in range(3):
            fb.filter_texture(plan, img, rho, N, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.fill_(1.0)
            a.record(stream)
            fb.filter_texture(plan, img, rho, N, out=out)
            b.record(stream)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        h_img = torch.from_numpy(f).pin_memory()
        h_out = torch.empty_like(h_img).pin_memory()
        t0 = time.perf_counter()
        for _ in range(steps):
            img.copy_(h_img, non_blocking=True)
            fb.filter_texture(plan, img, rho, N, out=out)
            h_out.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_s = (time.perf_counter() - t0) / steps
        px = B * H * W
        res[name] = {"Mpix/s": px / (ms * 1e-3) / 1e6, "ms": ms, "launches": plan.last_launch_count(),
                     "passes": 3, "e2e Mpix/s": px / e2e_s / 1e6, "e2e_ms": e2e_s * 1e3,
                     "h2d_bytes_per_call": 4 * px, "d2h_bytes_per_call": 4 * px,
                     "params": dict(fb.TEXTURE_DEFAULTS)}
    return res


def gauss_variant(fb, dev, flush, steps: int = 10):
    """NEXT-1: Algorithm 1 with the paper's Gaussian omega (eq.(4) on [-3 rho,
    3 rho]^2, fabf_filter_gauss): the classical filter of Table II (theta = f,
    sigma = 40) on 512x512 at rho = 3 / 5 / 10, N = 5 (the paper: 171-189 ms
    each on MATLAB / 3.4 GHz), and a 4K frame at rho = 5, N = 5.
    Synthetic Voronoi + noise images.  Device-timed."""
    import torch

    import workloads

    res = {}
    cases = [(512, 512, r, 5) for r in (3, 5, 10)] + [(2160, 3840, 5, 5)]
    for (H, W, rho, N) in cases:
        f = workloads.voronoi(H, W, seed=9000 + H, n_seeds=96, noise_sd=12.0).astype(np.float32)[None]
        img = torch.from_numpy(f).to(dev)
        sg = torch.full_like(img, 40.0)
        out = torch.empty_like(img)
        plan = fb.Plan(1, H, W)
        stream = torch.cuda.current_stream()
        for _ in range(3):
            fb.filter_gauss(plan, img, img, sg, rho, N, out=out)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            flush.fill_(1.0)
            a.record(stream)
            fb.filter_gauss(plan, img, img, sg, rho, N, out=out)
            b.record(stream)
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        res[f"gauss_{W}x{H}_rho{rho}_N{N}"] = {"Mpix/s": H * W / (ms * 1e-3) / 1e6, "ms": ms,
                                               "launches": plan.last_launch_count(),
                                               "fallback_pixels": plan.last_fallback_count()}
    return res


def run_sweep(args):
    """Config 5: 32 grey 1024^2 images, rho in {2,5,10,20,40} x N in {4,6,8,10},
    sigma ~ U[5,60], theta = f; one JSON line per (rho, N) cell with Mpix/s and
    the k_filter fp64 roofline fraction (cost should not depend on rho)."""
    import torch

    import paper_1811_02308_b200 as fb
    from paper_1811_02308_b200 import build
    import workloads

    build.build()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    gens = [g for g in args.sweep_generators.split(",") if g]
    for gen in gens:
        w0 = workloads.config5(2, 4, batch=32, size=1024, generator=gen)
        img = torch.from_numpy(w0.img).to(dev)
        th = torch.from_numpy(w0.theta).to(dev)
        sg = torch.from_numpy(w0.sigma).to(dev)
        out = torch.empty_like(img)
        plan = fb.Plan(*w0.shape)
        px = w0.img.size
        for rho in (2, 5, 10, 20, 40):
            for N in (4, 6, 8, 10):
                for _ in range(max(3, args.warmup)):
                    fb.filter(plan, img, th, sg, rho, N, out=out)
                stage = np.zeros(4)
                for i in range(args.steps):
                    flush.fill_(float(i))
                    _, ms4 = fb.filter_profile(plan, img, th, sg, rho, N, out=out)
                    stage += np.array(ms4)
                stage /= args.steps
                ms = float(stage.sum())
                kf = float(stage[2])
                mix = regime_mix(fb, plan, img, th, sg, rho, N)
                fl = alg_fp64_flops_per_pixel(N, mix["fp64_j"], mix["identity"]) * px / (kf * 1e-3) / 1e12
                print(json.dumps({"sweep": "config5", "generator": gen, "rho": rho, "N": N,
                                  "images": 32, "size": 1024, "value": px / (ms * 1e-3) / 1e6,
                                  "unit": "Mpix/s", "ms_per_step": ms,
                                  "stage_ms": {"k_bounds": stage[0] + stage[1], "k_filter": kf,
                                               "k_fallback": stage[3]},
                                  "fallback_pixels": plan.last_fallback_count(),
                                  "regime_mix": mix,
                                  "roofline": {"bound": "alu", "pipe": "fp64", "achieved": fl,
                                               "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                                               "frac": fl / FP64_PEAK_TFLOPS}}), flush=True)
    return 0


def run_band(args):
    """--shard band: ONE config-4 frame split into row bands over the ranks
    (strong scaling).  Every rank keeps its band of f, theta,
    sigma resident; a timed step is the halo exchange of rho rows of f with each
    neighbour (shard.exchange_halo: NCCL send / recv) plus fabf_filter on the
    band-plus-halo; the result stays on its rank.  Device time by CUDA events,
    max over ranks; value = the frame's pixels over that time."""
    import torch

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1811_02308_b200 as fb
    from paper_1811_02308_b200 import build, shard

    build.build()
    import workloads

    w = workloads.config(CFG)
    B, H, W = w.shape
    first, n = shard.band_shard(H, ws, rank, rho=w.rho)
    rows = slice(first, first + n)
    band = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, rows])).to(dev)
    f_b, th_b, sg_b = band(w.img), band(w.theta), band(w.sigma)
    f, th, sg, top = shard.band_problem(f_b, th_b, sg_b, w.rho, ws, rank)
    plan = fb.Plan(*f.shape)
    out = torch.empty_like(f)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    hl = f.shape[1] - n - top  # halo rows below

    def step():
        fh, _ = shard.exchange_halo(f_b, w.rho, ws, rank)  # the exchange step, every frame
        fb.filter(plan, fh, th, sg, w.rho, w.N, out=out)

    with ClockSampler(local) as clk:
        for i in range(max(3, args.warmup)):
            flush.fill_(float(i))
            step()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i, (a, b) in enumerate(ev):
            flush.fill_(float(i))
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
    tot_ms = shard.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), device=dev)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": B * H * W * args.steps / (tot_ms * 1e-3) / 1e6, "unit": "Mpix/s",
            "n_gpus": ws, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config 4, one frame in {ws} row bands (band_shard), rho-row halo of f exchanged "
                                   "with each neighbour every step (send/recv), no collective after filtering",
                       "rows_of_rank0": n, "halo_rows_above_below": [top, hl], "l2": "flushed between steps"},
            "gpu_launches": plan.last_launch_count() * args.steps,
            "halo_bytes_per_neighbour": 4 * w.rho * W * B, "clocks": clk.summary()}))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fabf", choices=["fabf", "reference"])
    ap.add_argument("--ref-pixels", type=int, default=0, help="oracle sample size (0: sized by --ref-seconds)")
    ap.add_argument("--ref-seconds", type=float, default=25.0, help="target oracle time for cpu_baseline")
    ap.add_argument("--sweep", action="store_true", help="config-5 (rho, N) sweep, one JSON line per cell")
    ap.add_argument("--sweep-generators", default="texture,rectangles")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer pass (launch-list captures)")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the configs 1-3 throughput lines")
    ap.add_argument("--shard", default="frames", choices=["frames", "band"],
                    help="N > 1: one frame per rank (weak, default) or one frame in row bands (strong)")
    args = ap.parse_args()
    if args.shard == "band" and args.impl == "fabf" and not args.sweep:
        return run_band(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.sweep:
        return run_sweep(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

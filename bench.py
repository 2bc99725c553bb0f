#!/usr/bin/env python
"""Benchmark of the B200 batch polynomial evaluator (BASELINE.json metric).

Default workload = BASELINE configs[3] (C4): trivariate sparse polynomial,
10,000 distinct terms (exponents 0..50 per variable), N(0,1) coefficients,
balanced scheme per variable, fp64, evaluated at 1e8 points U[-1,1]^3 — the
largest configuration that fits one GPU and the one the 8-GPU scaling target
is quoted on. One step = one evaluation of the whole 1e8-point batch.
Other configs: --config c1|c2|c3|c5 (each at its stated batch size).

  python bench.py [--gpus N --steps K --warmup W] [--config c4] [--impl reference]

Scaling is STRONG: the config's global batch is split into N contiguous
shards, one per rank (torchrun, NCCL for the barrier / max-reduction only; the
data path has no collective). Timing: CUDA events on the launching stream,
W untimed warm-up steps, K timed steps bracketed by barrier + synchronize,
max over ranks; value = global batch points / (max rank time per step).
L2 is flushed (256 MiB write) before every timed step.

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
the unmodified reference library through its Evaluator API, all host
threads, one session per thread) on the same workload: rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--points", type=int, default=0, help="override the global batch size")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--tune", default="", help="pe_tuning fields for every program, e.g. "
                    "iv_partition=3 (C5 through the one-pass split kernel); recorded in config")
    # plumbing check of the multi-rank path on a box with fewer GPUs than
    # ranks (tests/test_bench_ranks.py): every rank on cuda:0, gloo for the
    # barrier / max-reduction. Its numbers are not measurements.
    ap.add_argument("--ranks-share-gpu0", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


# ----------------------------------------------------------------- workloads

def workloads(cfg: str):
    from paper_1307_5655_b200 import workloads as W
    if cfg == "c2":
        return W.c2_all()
    return [W.ALL[cfg]()]


def metric_info(cfg: str):
    return {
        "c1": "C1: Horner dense d1000 fp64, 1e5 points U[-1,1] (launch-bound, parity case)",
        "c2": "C2: dense d1000 + d1023 fp64 U[-1,1], Estrin vs balanced, 1e7 points U[-1,1]",
        "c3": "C3: bivariate total-degree-40 int64 (861 terms), Horner/Horner, 1e7 points in [-2,2]^2",
        "c4": "C4: trivariate sparse 10k terms N(0,1), balanced x3, 1e8 points U[-1,1]^3",
        "c5": "C5: Estrin d200 interval, 1e8 intervals [x, x+1e-6]",
    }[cfg]


def shard(n_total: int, world: int, rank: int):
    """Contiguous shard [lo, lo + n) of the global batch for `rank`."""
    per = (n_total + world - 1) // world
    lo = min(n_total, rank * per)
    return lo, min(per, n_total - lo)


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 — clocks are evidence, not a dependency
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._nv is not None:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- ncu

# committed `ncu --set full` captures of the dominant kernels, taken at the
# bench's own per-launch sizes (scripts/ncu_captures.sh); a capture with
# several rows (the launches of one evaluate call) is summed
NCU_CAPTURES = {
    ("c4", "C4_trivariate_sparse10k"): "profiles/r2_ncu_c4_raw.csv",
    ("c5", "C5_interval_estrin_d200"): "profiles/r2_ncu_c5_raw.csv",
    # the one-pass split kernel (pe_tuning.iv_partition = 3)
    ("c5", "C5_interval_estrin_d200", "split"): "profiles/r2_ncu_c5_split_raw.csv",
    ("c2", "C2_estrin_d1000"): "profiles/r2_ncu_c2e1000_raw.csv",
    ("c2", "C2_balanced_d1000"): "profiles/r1_ncu_c2_balanced_d1000_raw.csv",
    ("c2", "C2_estrin_d1023"): "profiles/r1_ncu_c2_estrin_d1023_raw.csv",
    ("c2", "C2_balanced_d1023"): "profiles/r1_ncu_c2_balanced_d1023_raw.csv",
    ("c1", "C1_horner_d1000"): "profiles/r1_ncu_c1_raw.csv",
    ("c3", "C3_bivariate_td40_i64"): "profiles/r2_ncu_c3_raw.csv",
}


def ncu_traffic(cfg, program, points, variant=None):
    """(dram__bytes_read.sum + dram__bytes_write.sum per launch, source) from
    the committed ncu capture of this kernel; None when there is no capture
    at this launch size."""
    import csv
    path = NCU_CAPTURES.get((cfg, program, variant) if variant else (cfg, program))
    if not path or not os.path.exists(os.path.join(ROOT, path)):
        return None, None
    rows = list(csv.reader(open(os.path.join(ROOT, path))))
    head, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    for vals in rows[2:]:
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = head.index(name)
            total += float(vals[i]) * scale.get(units[i], 1)
    meta = os.path.join(ROOT, path.replace("_raw.csv", "_points.txt"))
    if os.path.exists(meta) and int(open(meta).read().split()[0]) != points:
        return None, f"{path} captured at a different size"
    return total, path


# ----------------------------------------------------------------- dist

def dist_setup(share_gpu0: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share_gpu0:
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if share_gpu0:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64,
                     device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------- CPU legs

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_kind():
    """("reference", host threads) when the unmodified reference library was
    built into oracle/_ref, else ("port", 1): the single-threaded C oracle."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if pyoracle.ref_available():
        return "reference", host_threads()
    return "port", 1


def _cpu_session(wl):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if pyoracle.ref_available():
        return pyoracle.Reference(wl.poly, wl.schemes)
    orc = pyoracle.Oracle(wl.poly, wl.schemes)

    class _Port:  # same call shape as Reference, threads ignored
        eval_f64 = staticmethod(lambda pts, t: orc.eval_f64(pts))
        eval_i64 = staticmethod(lambda pts, t: orc.eval_i64(pts))
        eval_interval = staticmethod(lambda lo, hi, t: orc.eval_interval(lo, hi))
    return _Port()


def cpu_reference_rate(wls, sample_points: int, threads: int):
    """points/s of the unmodified reference (oracle/_ref) on `threads` host
    threads, one Evaluator session per thread over contiguous shards (or of
    the C oracle port when the reference library is absent)."""
    total_pts, total_s = 0, 0.0
    for wl in wls:
        ref = _cpu_session(wl)
        if wl.domain == "interval":
            lo, hi = wl.points(sample_points)
            t = time.perf_counter()
            ref.eval_interval(lo, hi, threads)
        elif wl.domain == "i64":
            pts = wl.points(sample_points)
            t = time.perf_counter()
            ref.eval_i64(pts, threads)
        else:
            pts = wl.points(sample_points)
            t = time.perf_counter()
            ref.eval_f64(pts, threads)
        total_s += time.perf_counter() - t
        total_pts += sample_points
    return total_pts / total_s, total_s


def calibrate_sample(wls, threads, budget_s):
    rate, _ = cpu_reference_rate(wls, 64 * threads, threads)
    n = int(rate * budget_s)  # total points over all programs
    return max(threads * 16, n // len(wls))


def cpu_parallel_rate(wl, workers: int, points: int = 100):
    """The reference's intra-point threading (Evaluator::evaluate_parallel,
    eval.hpp:97-140) on `points` points, `workers` threads: points/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if not pyoracle.ref_available():
        return None
    ref = pyoracle.Reference(wl.poly, wl.schemes)
    pts = wl.points(points)
    if wl.domain == "interval":
        return points / ref.seconds_parallel_interval(pts[0], pts[1], workers)
    if wl.domain == "i64":
        return points / ref.seconds_parallel_i64(pts, workers)
    t = time.perf_counter()
    ref.eval_parallel_f64(pts, workers)
    return points / (time.perf_counter() - t)


def cpu_baseline(wls, seconds):
    kind, threads = cpu_kind()
    per = calibrate_sample(wls, threads, seconds)
    rate, secs = cpu_reference_rate(wls, per, threads)
    per1 = calibrate_sample(wls, 1, max(1.0, seconds / 6))
    rate1, secs1 = cpu_reference_rate(wls, per1, 1)
    par = cpu_parallel_rate(wls[0], threads)
    return {
        "value": rate, "unit": "points/s", "cores": threads, "kind": kind,
        "cpu_model": cpu_model(),
        "sample": f"{per} points per program x {len(wls)} programs ({secs:.1f} s), "
                  + ("unmodified reference Evaluator<D>, one session per thread"
                     if kind == "reference" else "C oracle port, 1 thread"),
        "single_thread": {"value": rate1, "unit": "points/s",
                          "sample": f"{per1} points per program ({secs1:.1f} s), 1 thread"},
        "evaluate_parallel": ({"value": par, "unit": "points/s", "workers": threads,
                               "sample": f"100 points of {wls[0].name}, reference "
                                         "Evaluator::evaluate_parallel (intra-point threads)"}
                              if par is not None else None),
    }


# ----------------------------------------------------------------- reference arm

def run_reference_arm(args, world, rank):
    wls = workloads(args.config)
    if rank != 0:
        return
    kind, threads = cpu_kind()
    per_step = calibrate_sample(wls, threads, budget_s=max(1.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_reference_rate(wls, per_step, threads)
    t0 = time.perf_counter()
    pts = 0
    for _ in range(args.steps):
        cpu_reference_rate(wls, per_step, threads)
        pts += per_step * len(wls)
    el = time.perf_counter() - t0
    value = pts / el
    terms = float(np.mean([wl.poly.coefficients.shape[0] for wl in wls]))
    line = {
        "impl": "reference",
        "metric": "points/s", "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": {"c3": "int64", "c5": "f64-interval"}.get(args.config, "f64"),
        "data": "synthetic (seeded PCG64, explicit transforms)",
        "config": {"workload": metric_info(args.config), "programs": [w.name for w in wls],
                   "points_per_step": per_step * len(wls)},
        "term_evals_per_s": value * terms,
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads,
                         "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{per_step} points per program per step, {len(wls)} programs, "
                                   + ("unmodified reference Evaluator<D>, one session per thread"
                                      if kind == "reference" else "C oracle port, 1 thread")},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- native arm

def run_native(args, world, rank, local):
    import torch
    import paper_1307_5655_b200 as pe

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    wls = workloads(args.config)
    n_total = args.points or wls[0].n_points
    lo_idx, n = shard(n_total, world, rank)
    domain = wls[0].domain

    # programs + kernels (compile is setup, outside the timed region)
    t_setup = time.perf_counter()
    progs = [pe.compile(w.poly, w.schemes) for w in wls]
    tune = {k.strip(): int(v) for k, v in (kv.split("=") for kv in args.tune.split(",") if kv)}
    for p in progs:
        if tune:
            p.set_tuning(**tune)
    if domain == "interval":
        evs = [pe.Evaluator(pe.IntervalDomain(), p, device=local, deferred_checks=True)
               for p in progs]
    elif domain == "i64":
        evs = [pe.Evaluator(pe.BigIntDomain(), p, device=local, deferred_checks=True)
               for p in progs]
    else:
        evs = [pe.Evaluator(pe.DoubleDomain(), p, device=local) for p in progs]

    # this rank's contiguous shard of the global batch (seeded per shard)
    if domain == "interval":
        lo, hi = wls[0].points(n, offset_tag=rank)
        inputs = ([torch.from_numpy(a).to(dev) for a in lo], [torch.from_numpy(a).to(dev) for a in hi])
        host_arrays = (lo, hi)
        outs = [(torch.empty(n, dtype=torch.float64, device=dev),
                 torch.empty(n, dtype=torch.float64, device=dev)) for _ in wls]
        bytes_in = 16 * n * wls[0].poly.nvars
        bytes_out = 16 * n
    else:
        pts = wls[0].points(n, offset_tag=rank)
        inputs = [torch.from_numpy(a).to(dev) for a in pts]
        host_arrays = pts
        dt = torch.int64 if domain == "i64" else torch.float64
        outs = [torch.empty(n, dtype=dt, device=dev) for _ in wls]
        bytes_in = 8 * n * wls[0].poly.nvars
        bytes_out = 8 * n
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    for e, o in zip(evs, outs):  # first call: walk VM while the kernel compiles
        e.evaluate(inputs, out=o, stream=sptr)
    torch.cuda.synchronize(dev)
    first_result_s = time.perf_counter() - t_setup
    # wait for the specialised kernels (background compile) before timing
    dom_codes = {"f64": [pe.DOMAIN_F64], "interval": [pe.DOMAIN_INTERVAL],
                 "i64": [pe.DOMAIN_I64F, pe.DOMAIN_I64]}[domain]
    for p in progs:
        for dc in dom_codes:
            p.compile_only(dc)
    for e, o in zip(evs, outs):
        e.evaluate(inputs, out=o, stream=sptr)
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup

    # FP64 / int64-MAD pipe peak on this GPU (roofline denominator)
    import ctypes as C
    from paper_1307_5655_b200 import _lib as L
    int_tier = "fp64-exact"
    if domain == "i64":
        _, b53 = progs[0].i64_bounds()
        coord_max = [int(t.abs().max().item()) for t in inputs]
        if not all(m <= b for m, b in zip(coord_max, b53)):
            int_tier = "int64-imad"
    peak, sms = C.c_double(), C.c_int32()
    L.check(L.lib().pe_measure_peak(local, 1 if int_tier == "int64-imad" else 0,
                                    C.byref(peak), C.byref(sms)))
    int_peak = C.c_double()
    if domain == "i64":
        L.check(L.lib().pe_measure_peak(local, 1, C.byref(int_peak), C.byref(sms)))

    # L2 flush buffer (> 126 MB L2) written between timed steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(events=None):
        for i, (e, o) in enumerate(zip(evs, outs)):
            if events is not None:
                events[i][0].record(stream)
            e.evaluate(inputs, out=o, stream=sptr)
            if events is not None:
                events[i][1].record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    launches0 = pe.launch_count()
    per_launch_ms = [[] for _ in wls]
    t_total = 0.0
    # The K steps are bracketed as a whole by barrier + synchronize; inside,
    # every step is enqueued back to back (L2 flush outside the step's event
    # pair, then the evaluate calls), so no step's events include the GPU
    # idling for the host.
    with ClockSampler(torch.cuda.current_device()) as clocks:
        barrier(world)
        torch.cuda.synchronize(dev)
        all_ev = []
        for _ in range(args.steps):
            flush.zero_()  # outside the timed interval: L2 cold at each step
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in wls]
            step(ev)
            all_ev.append(ev)
        torch.cuda.synchronize(dev)
        barrier(world)
    for e in evs:  # deferred domain checks (int64 bound, interval endpoints)
        if getattr(e, "deferred_checks", False):
            e.synchronize(sptr)
    for ev in all_ev:
        ms = [a.elapsed_time(b) for a, b in ev]
        for i, m in enumerate(ms):
            per_launch_ms[i].append(m)
        t_total += ev[0][0].elapsed_time(ev[-1][1])
    launches = pe.launch_count() - launches0
    t_total = max_over_ranks(t_total, world)
    ms_step = t_total / args.steps
    pts_step = n_total * len(wls)  # the global batch, all ranks
    value = pts_step / (ms_step * 1e-3)

    # roofline of the dominant kernel (longest average launch)
    avg = [statistics.mean(x) for x in per_launch_ms]
    top = int(np.argmax(avg))
    st = progs[top].kernel_stats(
        {"f64": pe.DOMAIN_F64, "i64": pe.DOMAIN_I64, "interval": pe.DOMAIN_INTERVAL}[domain])
    info = progs[top].info()
    if domain == "f64":
        algo_per_pt = info["walk_muls"] + info["power_muls"]
        unit_ops = "DFMA"
    elif domain == "i64":
        algo_per_pt = info["walk_muls"] + info["power_muls"]  # int64 MADs (adds fused)
        unit_ops = ("exact DFMA (int64 MAD on the FP64 pipe)" if int_tier == "fp64-exact"
                    else "int64 MAD")
    else:
        algo_per_pt = 2 * info["walk_adds"] + 4 * (info["walk_muls"] + info["power_muls"])
        unit_ops = "fp64 add/mul (interval endpoints)"
    achieved = algo_per_pt * n / (avg[top] * 1e-3)  # FP64-pipe ops/s (or int64 MAD/s)
    nominal = sms.value * 64 * 1.965e9
    fp_pipe = domain != "i64" or int_tier == "fp64-exact"
    # FLOP accounting: a DFMA is 2 FLOP, an interval endpoint add/mul 1; the
    # FP64 pipe issues one of either per lane per clock
    flop_per_op = 1.0 if domain == "interval" else 2.0
    sections = progs[top].f64_slices() if domain == "f64" else 1
    kernel_name = f"pe_walk_{domain} [{wls[top].name}]"
    if domain == "f64" and sections > 1:
        kernel_name = (f"pe_walk_f64 [{wls[top].name}]: one persistent kernel, {sections} sections "
                       "(pe_section0..) over groups of 4 tiles")
    iv_ptx = progs[top].ptx(pe.DOMAIN_INTERVAL) if domain == "interval" else ""
    if "pe_walk_interval_split" in iv_ptx:
        kernel_name = (f"pe_walk_interval_split + pe_walk_interval_fix [{wls[top].name}] (one "
                       "evaluate call: one-pass sign split, then the fixup replay)")
    elif "pe_walk_interval_pos" in iv_ptx:
        kernel_name = (f"classify_intervals + pe_walk_interval_pos + pe_walk_interval_neg + "
                       f"pe_walk_interval_fix [{wls[top].name}] (one evaluate call, sign-partitioned)")
    traffic, traffic_src = ncu_traffic(args.config, wls[top].name, n,
                                       "split" if "pe_walk_interval_split" in iv_ptx else None)
    roofline = {
        "bound": "fp64" if fp_pipe else "int64_mad",
        "int64_tier": int_tier if domain == "i64" else None,
        "frac_vs_int64_mad_peak": (achieved / int_peak.value) if domain == "i64" else None,
        "achieved": (achieved * flop_per_op / 1e12) if fp_pipe else achieved / 1e12,
        "peak": (peak.value * flop_per_op / 1e12) if fp_pipe else peak.value / 1e12,
        "unit": "TFLOP/s" if fp_pipe else "T int64-MAD/s",
        "frac": achieved / peak.value,
        "frac_vs_nominal": achieved / nominal if fp_pipe else None,
        "achieved_pipe_ops_per_s": achieved, "peak_pipe_ops_per_s": peak.value,
        "peak_source": "measured live: pe_measure_peak microbenchmark (8 independent chains/thread, "
                       "full occupancy, immediate multiplier, best of 16 after 16 warm-up launches) "
                       "on this GPU; nominal FP64 FMA pipe = "
                       f"{nominal / 1e12:.1f} T DFMA/s at 1965 MHz x {sms.value} SMs x 64 lanes "
                       "(MEASURED_PEAKS.json has no FP64 entry)",
        "ops": f"{algo_per_pt} {unit_ops} per point (SURVEY 8d F) x {n} points per launch",
        "kernel": kernel_name,
        "issued_fp64_per_point": st["fp_ops"], "issued_int64_per_point": st["int_ops"],
        "hbm_frac": (bytes_in + bytes_out) / (avg[top] * 1e-3) / 1e9 /
                    json.load(open(MEASURED))["hbm_gbs"] if os.path.exists(MEASURED) else None,
        "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_bytes_per_launch": bytes_in + bytes_out,
        "per_program_ms": {w.name: round(a, 4) for w, a in zip(wls, avg)},
    }

    # e2e through the public API with HOST buffers: H2D + walk + D2H in the
    # timed region, pinned (page-locked) and pageable (plain numpy) inputs
    e2e = None
    if not args.no_e2e:
        multi = domain == "f64" and len(progs) > 1

        def host_call(hin, hout):
            if multi:
                pe.evaluate_many(progs, hin, outs=hout, device=local)
                return
            for e, o in zip(evs, hout):
                e.evaluate(hin, out=o)

        def timed(hin, hout, steps):
            host_call(hin, hout)
            barrier(world)
            t0 = time.perf_counter()
            for _ in range(steps):
                host_call(hin, hout)
            el = max_over_ranks(time.perf_counter() - t0, world)
            return pts_step / (el / steps)

        k = max(1, args.steps // 4)
        if domain == "interval":
            pin_in = (tuple(torch.from_numpy(a).pin_memory().numpy() for a in host_arrays[0]),
                      tuple(torch.from_numpy(a).pin_memory().numpy() for a in host_arrays[1]))
            pin_out = [(torch.empty(n, dtype=torch.float64).pin_memory().numpy(),
                        torch.empty(n, dtype=torch.float64).pin_memory().numpy()) for _ in wls]
            pag_in = (tuple(np.array(a) for a in host_arrays[0]), tuple(np.array(a) for a in host_arrays[1]))
            pag_out = [(np.empty(n), np.empty(n)) for _ in wls]
        else:
            dt = torch.int64 if domain == "i64" else torch.float64
            pin_in = [torch.from_numpy(a).pin_memory().numpy() for a in host_arrays]
            pin_out = [torch.empty(n, dtype=dt).pin_memory().numpy() for _ in wls]
            pag_in = [np.array(a) for a in host_arrays]
            pag_out = [np.empty(n, dtype=np.int64 if domain == "i64" else np.float64) for _ in wls]
        v_pin = timed(pin_in, pin_out, k)
        v_pag = timed(pag_in, pag_out, k)
        e2e = {"value": v_pin, "unit": "points/s",
               "h2d_bytes_per_step": bytes_in * (1 if multi else len(wls)) * world,
               "d2h_bytes_per_step": bytes_out * len(wls) * world,
               "path": ("pe_eval_f64_multi" if multi else "pe_eval_*")
                       + " with page-locked host buffers (chunked H2D / walk / D2H pipeline)",
               "pageable": {"value": v_pag, "unit": "points/s",
                            "path": "same call with plain numpy (pageable) buffers: host threads "
                                    "copy through page-locked staging slots"},
               "steps": k}

    # CPU baseline: the unmodified reference on this box's host cores (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(wls, args.cpu_seconds)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "points/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    terms = float(np.mean([wl.poly.coefficients.shape[0] for wl in wls]))
    line = {
        "metric": "points/s", "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": {"c3": "int64", "c5": "f64-interval"}.get(args.config, "f64"),
        "data": "synthetic (seeded PCG64, explicit transforms; SURVEY 8d)",
        "config": {"workload": metric_info(args.config), "programs": [w.name for w in wls],
                   "global_batch": n_total, "points_per_rank": n, "point_evals_per_step": pts_step,
                   "parallelism": f"global batch in {world} contiguous shard(s), one per rank, "
                                  "no data-path collective",
                   "l2": "flushed (256 MiB write) before every timed step",
                   **({"tuning": tune} if tune else {})},
        "term_evals_per_s": value * terms,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks.summary(),
        "setup_s": setup_s,
        "first_result_s": first_result_s,
        "setup_note": "first_result_s: compile + first evaluate of the shard (walk VM while the "
                      "specialised kernel compiles in the background); setup_s: until the "
                      "specialised kernel is compiled, loaded and has run once",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs it, other ranks exit without work
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, world, rank)
        return
    world, rank, local = dist_setup(args.ranks_share_gpu0)
    try:
        run_native(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

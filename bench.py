"""bench.py -- BASELINE metric on the B200: AB-join distance cells/s (GCell/s)
and % of the FP64 roofline, next to the reference CPU join.

Workload (BASELINE.json configs[3], "C4"): a 2^24-sample random-walk query
(seed 4) joined against a dictionary of 256 random-walk segments x 1024
samples (seed 5), m = 512, FP64 -- the config the north-star target is quoted
on. One step = one full dictionary join of the query: window statistics +
the join kernel + epilogue, inputs resident in HBM. Inputs are seeded
synthetic data with the BASELINE shapes (no dataset needed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

The same JSON line also carries every other BASELINE config ("configs": C1,
C2, C3, C5 and C4 in the FP32 mode; inputs from workloads.py), each with its
device time, roofline fraction and a same-run CPU baseline of the reference
itself, plus the self-join target shape (2^21 x m = 512).

N > 1: weak scaling -- every rank joins its own C4 query (seed 4 + rank)
against the same dictionary; no collective on the data path (rows are
independent). Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

Q_LEN = 1 << 24
N_SEG = 256
SEG_LEN = 1024
M = 512
Q_SEED, D_SEED = 4, 5
FLOPS_PER_CELL = 6  # profiles.hpp:330-331: 2 mul + 2 add (update) + 2 mul (normalise)
CPU_SAMPLE_WINDOWS = 1 << 17  # bounded CPU-baseline sample of C4 (query windows; 2^17-2^18)


def cells_per_step(q_len=Q_LEN):
    return (q_len - M + 1) * N_SEG * (SEG_LEN - M + 1)


def workload_config():
    return {"workload": "C4: FP64 dictionary AB-join, random-walk query 2^24 (seed 4) vs 256 random-walk segments "
                        "x 1024 (seed 5), m=512, straddling windows masked",
            "query_len": Q_LEN, "segments": N_SEG, "segment_len": SEG_LEN, "m": M,
            "cells_per_step": cells_per_step(),
            "l2": "query (128 MiB) + window stats exceed the 126 MB L2; L2 flushed with a 256 MiB write between steps"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region"""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and "Active" in r[3 + k]
                          and "Not" not in r[3 + k]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- inputs
def make_dictionary():
    from paper_2112_12965_b200 import synth
    import paper_2112_12965_b200 as tsd
    segs = synth.walks(D_SEED, N_SEG, SEG_LEN)
    return tsd.Dictionary([tsd.Segment(SEG_LEN * s, segs[s]) for s in range(N_SEG)], m=M,
                          source_length=N_SEG * SEG_LEN), segs


def make_query(seed):
    from paper_2112_12965_b200 import synth
    return synth.walk(seed, Q_LEN)


# ---------------------------------------------------------------- CPU baseline (reference)
def cpu_reference_gcells(q, segs, threads, windows=CPU_SAMPLE_WINDOWS):
    """the unmodified reference join_dictionary (oracle/_ref) on the first
    `windows` query windows, all host threads; falls back to the plain-C port
    (single thread) when the reference build is absent"""
    from oracle import py_oracle as O
    sub = q[: windows + M - 1]
    t0 = time.perf_counter()
    if O.ref_available():
        O.ref_join_dictionary(sub, list(segs), [SEG_LEN * s for s in range(N_SEG)], M, threads=threads)
        kind, cores = "reference", threads
    else:
        O.dict_join(sub, list(segs), [SEG_LEN * s for s in range(N_SEG)], M)
        kind, cores = "port", 1
    dt = time.perf_counter() - t0
    cells = windows * N_SEG * (SEG_LEN - M + 1)
    return {"value": cells / dt / 1e9, "unit": "GCell/s", "cores": cores, "kind": kind,
            "sample": f"first {windows} query windows of C4 x all 256 segments ({cells:.3e} cells, {dt:.1f} s)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _timed(fn, reps=1):
    """best-of-reps wall time of fn() (the reference bench's rule, tools/tsdict.cpp:219-230)"""
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    _, segs = make_dictionary()
    q = make_query(Q_SEED)
    threads = os.cpu_count() or 1
    vals = []
    windows = args.ref_windows or (1 << 15)
    for s in range(args.warmup + args.steps):
        r = cpu_reference_gcells(q, segs, threads, windows=windows)
        if s >= args.warmup:
            vals.append(r["value"])
        if s == 0 and not args.ref_windows:
            # size the sample from the first warm-up step: the largest power of
            # two up to 2^17 windows (BASELINE.md section 3's prefix) that keeps
            # the whole run near 150 s; longer prefixes amortise the reference's
            # per-call thread start-up, so they are the fairer figure
            dt = (1 << 15) * N_SEG * (SEG_LEN - M + 1) / (r["value"] * 1e9)
            rest = max(1, args.warmup + args.steps - 1)
            while windows < (1 << 17) and rest * dt * (2 * windows / (1 << 15)) <= 150.0:
                windows *= 2
    v = statistics.median(vals)
    cb = dict(r, value=v)
    line = {"impl": "reference", "metric": "AB-join distance cells/sec", "value": v, "unit": "GCell/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cells_per_step() / (v * 1e9) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random walks, BASELINE C4 shapes)",
            "config": dict(workload_config(), note="each step times the reference on a bounded sample of the "
                                                  "workload; ms_per_step extrapolates to the full step"),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "GCell/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import paper_2112_12965_b200 as tsd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    D, segs = make_dictionary()
    q = make_query(Q_SEED + rank)
    nrows = Q_LEN - M + 1
    plan = tsd.DictPlan(D, M)
    d_q = torch.from_numpy(q).to(dev)
    d_val = torch.empty(nrows, dtype=torch.float64, device=dev)
    d_idx = torch.empty(nrows, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.join_device(d_q.data_ptr(), [Q_LEN], d_val.data_ptr(), d_idx.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    launches = 0
    join_ms, kernel_ms, heads_ms = [], [], []
    elapsed_ms = 0.0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between steps (not timed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            elapsed_ms += e0.elapsed_time(e1)
            s_ms, j_ms, nl = plan.last_timing()
            k_ms, h_ms = plan.last_kernel_timing()
            join_ms.append(j_ms)
            kernel_ms.append(k_ms)
            heads_ms.append(h_ms)
            launches += nl
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    total_cells = cells_per_step() * world * args.steps
    value = total_cells / (elapsed_ms * 1e-3) / 1e9

    # end to end through the reference-facing C ABI (host buffers, pinned)
    h_q = torch.from_numpy(q).pin_memory()
    h_val = torch.empty(nrows, dtype=torch.float64).pin_memory()
    h_idx = torch.empty(nrows, dtype=torch.int64).pin_memory()
    seg_all = np.ascontiguousarray(np.concatenate(list(segs)))
    lib = tsd.load_library()
    import ctypes
    lens = np.full(N_SEG, SEG_LEN, dtype=np.uintp)
    starts = np.arange(N_SEG, dtype=np.uintp) * SEG_LEN
    f64p, i64p, szp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_size_t)

    def e2e_call():
        rc = lib.tsd_dict_join(ctypes.cast(h_q.data_ptr(), f64p), Q_LEN, seg_all.ctypes.data_as(f64p),
                               lens.ctypes.data_as(szp), starts.ctypes.data_as(szp), N_SEG, M, 0,
                               ctypes.cast(h_val.data_ptr(), f64p), ctypes.cast(h_idx.data_ptr(), i64p))
        if rc:
            raise RuntimeError(lib.tsd_last_error().decode())

    e2e_call()  # warm (thread context, arena)
    e2e_steps = max(1, min(args.steps, 3))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = cells_per_step() * world / e2e_s / 1e9
    # sanity: the e2e result equals the device-resident result
    same = bool(torch.equal(h_idx, d_idx.cpu())) and bool(torch.equal(h_val, d_val.cpu()))

    plan.close()  # release the FP64 plan's device arenas before the FP32 plan
    del h_q, h_val, h_idx
    fp32 = fp32_line(D, d_q, d_val, d_idx, stream, flush, dev, dist, world)
    del d_q, d_val, d_idx
    torch.cuda.empty_cache()
    sj = self_join_lines(q, dist, world)  # every rank (the sharded run needs all of them)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    peak_meas, peak_mhz = tsd.measure_peak_clock("fp64", seconds=2.0)
    nominal = nominal_peaks(dev, clk.summary())
    peak = nominal["fp64"]
    for v in sj.values():  # against the FP64 cell peak of the GPUs used
        v["frac_of_fp64_cell_peak"] = v["value"] * 1e9 / (v.get("n_gpus", 1) * peak / FLOPS_PER_CELL)
        if v.get("kernel_ms"):
            v["kernel_frac"] = FLOPS_PER_CELL * v["pairs"] / (v["kernel_ms"] * 1e-3) / peak
    fp32["roofline"]["peak_measured"] = fp32["roofline"]["peak"]
    fp32["roofline"]["peak"] = nominal["fp32"] / 1e12
    fp32["roofline"]["frac_of_measured"] = fp32["roofline"]["frac"]
    fp32["roofline"]["frac"] = fp32["roofline"]["achieved"] * 1e12 / nominal["fp32"]
    fp32["roofline"]["peak_def"] = ("nominal FFMA peak: %d SMs x 128 lanes x 2 flops x %.0f MHz (max SM clock); "
                                    "peak_measured: FFMA loop measured live" % (nominal["sms"], nominal["mhz"]))
    configs = config_lines(args, dev, stream, flush, peak, nominal)
    jms = statistics.median(join_ms)
    kms = statistics.median(kernel_ms)
    hms = statistics.median(heads_ms)
    achieved = FLOPS_PER_CELL * cells_per_step() / (kms * 1e-3)
    if args.traffic is not None:
        traffic, traffic_src = args.traffic, "--traffic argument"
    else:
        traffic, traffic_src = measure_traffic()
        if traffic is None:
            why = traffic_src
            traffic = committed_traffic()
            traffic_src = ("committed ncu capture (profiles/r1_k_join_traffic.json); in-run measurement: " + why
                           if traffic is not None else why)
    roofline = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_measured": peak_meas / 1e12, "frac_of_measured": achieved / peak_meas,
                "peak_measured_sm_mhz": peak_mhz,
                "kernel": "k_join<8,false,false> (FP64 row-band join)", "achieved_def":
                    "6 FP64 flops per valid cell (profiles.hpp:330-331) x cells per launch / median duration of "
                    "the join kernel (CUDA events around its launch, on the launching stream)",
                "traffic_def": "dram__bytes_read.sum + dram__bytes_write.sum of one k_join launch",
                "traffic_source": traffic_src,
                "algorithmic_bytes": algo_bytes_per_launch(),
                "pipeline": {"join_ms_median": jms, "kernel_ms_median": kms, "heads_fft_ms_median": hms,
                             "frac": FLOPS_PER_CELL * cells_per_step() / (jms * 1e-3) / peak,
                             "def": "the whole join phase (column packing, FFT heads, join kernel, group merge)"},
                "peak_def": "nominal DFMA peak: %d SMs x 64 FP64 FMA/clk x 2 flops x %.0f MHz (max SM clock; "
                            "MEASURED_PEAKS.json has no FP64 entry); peak_measured: a DFMA loop timed live on this "
                            "GPU for 2 s (tsd_measure_peak_clock, SM clock it ran at: peak_measured_sm_mhz)"
                            % (nominal["sms"], nominal["mhz"])}
    cpu = cpu_reference_gcells(q, segs, os.cpu_count() or 1) if world == 1 or rank == 0 else None
    if cpu:
        cpu["cpu_model"] = cpu_model()
        cpu["extrapolated"] = True
    line = {"metric": "AB-join distance cells/sec", "value": value, "unit": "GCell/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded random walks with the BASELINE C4 shapes)", "config": workload_config(),
            "parallelism": f"weak x{world}: one C4 query per GPU, shared dictionary, no data-path collective",
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GCell/s", "h2d_bytes_per_step": int(Q_LEN * 8 + seg_all.nbytes),
                    "d2h_bytes_per_step": int(nrows * 16), "api": "tsd_dict_join (host buffers, pinned)",
                    "matches_device_path": same},
            "gpu_launches": launches, "clocks": clk.summary(),
            "fp32": fp32,
            "self_join": sj,
            "configs": configs,
            "join_ms_median": jms, "fraction_of_fp64_peak_cells": (cells_per_step() / (jms * 1e-3)) /
                                                                    (peak / FLOPS_PER_CELL)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def fp32_line(D, d_q, d_val, d_idx, stream, flush, dev, dist=None, world=1, steps=3, warmup=3):
    """BASELINE C4 in the optional FP32 mode (north star: distances within
    1e-3 absolute): the same device-resident step, with the join kernel's
    achieved fraction of the FP32 cell roofline (6 FP32 flops per cell at the
    FFMA peak measured live). Timed like the FP64 line (CUDA events on the
    launching stream, L2 flushed between steps, max over ranks)."""
    import torch
    import paper_2112_12965_b200 as tsd
    plan = tsd.DictPlan(D, M, "fp32")

    def step():
        plan.join_device(d_q.data_ptr(), [Q_LEN], d_val.data_ptr(), d_idx.data_ptr(), stream.cuda_stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    ms, kms = 0.0, []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        kms.append(plan.last_kernel_timing()[0])
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    plan.close()
    peak32 = tsd.measure_peak("fp32", seconds=1.0)
    k = statistics.median(kms)
    return {"value": cells_per_step() * world * steps / (ms * 1e-3) / 1e9, "unit": "GCell/s",
            "ms_per_step": ms / steps, "dtype": "f32 sweep, FP64 statistics / heads / final correlation",
            "roofline": {"bound": "fp32", "achieved": FLOPS_PER_CELL * cells_per_step() / (k * 1e-3) / 1e12,
                         "peak": peak32 / 1e12, "unit": "TFLOP/s",
                         "frac": FLOPS_PER_CELL * cells_per_step() / (k * 1e-3) / peak32,
                         "kernel": "k_join<16,false,true> (FP32 f32x2 row-band join)",
                         "peak_def": "FFMA throughput measured live by tsd_measure_peak (1 s, this GPU)"}}


def self_join_lines(q, dist=None, world=1):
    """Self-join throughput in the reference's unit (one admissible unordered
    pair |i - j| > excl evaluated once, profiles.hpp:287-297):
    the SURVEY's proposed target (a 2^21 prefix of the C4 query, m = 512,
    excl = m/2) and BASELINE C2 (ECG-like, n = 131072, m = 250, excl = m/4).
    Host API (tsd_self_join), so host<->device copies are inside the time.
    N > 1 (torchrun): the sharded self-join over all ranks -- strong scaling,
    one all-gather of per-row partials, max-over-ranks time. Call on every
    rank; the frac fields are added by the caller."""
    import torch
    import paper_2112_12965_b200 as tsd
    from paper_2112_12965_b200 import synth
    out = {}
    if dist is not None and world > 1:
        # opt-in (TSD_BENCH_SHARDED_SELF=1): the NCCL path of the sharded
        # self-join has only run on one GPU and under gloo so far, and a fault
        # in this side line must not cost the scaling run its headline
        if os.environ.get("TSD_BENCH_SHARDED_SELF", "0") != "1":
            return out
        x = np.ascontiguousarray(q[: 1 << 21])
        m = 512
        cnt, e = x.size - m + 1, m // 2
        pairs = (cnt - e - 1) * (cnt - e) / 2
        tsd.self_join_sharded(x, m)  # warm
        ts = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tsd.self_join_sharded(x, m)
            torch.cuda.synchronize()
            t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t.item()))
        t = statistics.median(ts)
        out["self_2^21_m512_sharded"] = {"n": int(x.size), "m": m, "excl": e, "pairs": pairs, "ms": t * 1e3,
                                         "value": pairs / t / 1e9, "unit": "GPair/s", "n_gpus": world,
                                         "scaling": "strong",
                                         "kernel": "symmetric upper-triangle sweep, sharded by task + all-gather"}
        return out
    for name, x, m, excl in (("self_2^21_m512", np.ascontiguousarray(q[: 1 << 21]), 512, None),
                             ("C2_self_ecg_m250", synth.ecg(2, 131072)[0], 250, 62)):
        cnt = x.size - m + 1
        e = m // 2 if excl is None else excl
        pairs = (cnt - e - 1) * (cnt - e) / 2
        tsd.self_join(x, m, excl=excl)  # warm
        ts, dms, kms = [], [], []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tsd.self_join(x, m, excl=excl)
            ts.append(time.perf_counter() - t0)
            d_ms, k_ms, _ = tsd.last_join_timing()
            dms.append(d_ms)
            kms.append(k_ms)
        t = statistics.median(ts)
        if os.environ.get("TSD_BENCH_DEBUG"):
            print(f"[bench] {name}: {[round(v * 1e3, 2) for v in ts]} ms", file=sys.stderr, flush=True)
        out[name] = {"n": int(x.size), "m": m, "excl": e, "pairs": pairs, "ms": t * 1e3,
                     "value": pairs / t / 1e9, "unit": "GPair/s",
                     "device_ms": statistics.median(dms), "kernel_ms": statistics.median(kms),
                     "timing": "ms / value: host API wall time incl. copies (median of 5); device_ms: CUDA events "
                               "from window statistics to epilogue; kernel_ms: the main sweep kernel",
                     "kernel": "symmetric upper-triangle sweep" if (m >= 192 and cnt >= max(98304, (1 << 26) // m))
                     else "full-matrix sweep"}
    return out


def nominal_peaks(dev, clocks):
    """nominal FMA-pipe peaks of this GPU at its maximum SM clock (B200: 64
    FP64 and 128 FP32 FMA lanes per SM per clock)"""
    import torch
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mhz = clocks.get("sm_max_mhz") or 1965.0
    return {"sms": sms, "mhz": mhz, "fp64": sms * 64 * 2 * mhz * 1e6, "fp32": sms * 128 * 2 * mhz * 1e6}


def _event_steps(step, stream, flush, steps, warmup, after=None):
    """CUDA-event time (ms) of each of `steps` calls of step() on `stream`,
    after `warmup` untimed calls, L2 flushed before each (not timed)"""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    out = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
        if after:
            after()
    return out


def _plan_config(cfg, series, dev, stream, flush, peak, steps=5, warmup=3):
    """device-resident dictionary join of `series` (list of 1-D arrays) on a
    plan of cfg's dictionary: (ms per step, join kernel ms, launches)"""
    import torch
    import paper_2112_12965_b200 as tsd
    import workloads as W
    m = cfg["m"]
    plan = tsd.DictPlan(W.dictionary(cfg), m)
    lens = [len(x) for x in series]
    d_q = torch.from_numpy(np.ascontiguousarray(np.concatenate(series))).to(dev)
    rows = sum(n - m + 1 for n in lens)
    d_val = torch.empty(rows, dtype=torch.float64, device=dev)
    d_idx = torch.empty(rows, dtype=torch.int64, device=dev)
    kms, nl = [], []

    def step():
        plan.join_device(d_q.data_ptr(), lens, d_val.data_ptr(), d_idx.data_ptr(), stream.cuda_stream)

    def after():
        kms.append(plan.last_kernel_timing()[0])
        nl.append(plan.last_timing()[2])
    ms = _event_steps(step, stream, flush, steps, warmup, after)
    plan.close()
    return statistics.median(ms), statistics.median(kms), nl[-1]


def _frac(cells, ms, peak):
    return FLOPS_PER_CELL * cells / (ms * 1e-3) / peak


def config_lines(args, dev, stream, flush, peak, nominal):
    """BASELINE configs C1, C2, C3, C5 (workloads.py) on this GPU, each with a
    same-run CPU baseline of the unmodified reference (oracle/_ref, all host
    threads). value = cells (pairs) per second of the device step."""
    import torch
    import paper_2112_12965_b200 as tsd
    import workloads as W
    from oracle import py_oracle as O
    if args.skip_configs:
        return None
    threads = os.cpu_count() or 1
    model = cpu_model()
    have_ref = O.ref_available()
    out = {}

    def cpu_line(value, unit, sample, extrapolated, kind="reference"):
        return {"value": value, "unit": unit, "cores": threads, "cpu_model": model, "kind": kind,
                "sample": sample, "extrapolated": extrapolated}

    # ---- C1: exact AB-join against 8 x 512, m = 100 (launch-bound: 5.4e7 cells)
    c = W.c1()
    ms, kms, nl = _plan_config(c, [c["q"]], dev, stream, flush, peak, steps=20)
    line = {"workload": "C1: walk 16384 (seed 0) vs 8 walks x 512 (seed 1), m=100, FP64", "cells": c["cells"],
            "ms": ms, "kernel_ms": kms, "value": c["cells"] / (ms * 1e-3) / 1e9, "unit": "GCell/s",
            "frac": _frac(c["cells"], kms, peak), "gpu_launches_per_step": nl}
    if have_ref:
        dt = _timed(lambda: O.ref_join_dictionary(c["q"], c["segs"], c["starts"], c["m"], threads=threads), 3)
        line["cpu_baseline"] = cpu_line(c["cells"] / dt / 1e9, "GCell/s", "full run, best of 3", False)
    out["C1"] = line

    # ---- C2: self-join, ECG n = 131072, m = 250, excl = m/4
    c = W.c2()
    tsd.self_join(c["t"], c["m"], excl=c["excl"])
    hs, ds, ks = [], [], []
    for _ in range(5):
        t0 = time.perf_counter()
        tsd.self_join(c["t"], c["m"], excl=c["excl"])
        hs.append((time.perf_counter() - t0) * 1e3)
        d_ms, k_ms, nl = tsd.last_join_timing()
        ds.append(d_ms)
        ks.append(k_ms)
    dms, kms = statistics.median(ds), statistics.median(ks)
    line = {"workload": "C2: self-join, ECG-like n=131072 (seed 2), m=250, excl=m/4=62, FP64", "pairs": c["pairs"],
            "ms": dms, "kernel_ms": kms, "host_api_ms": statistics.median(hs),
            "value": c["pairs"] / (dms * 1e-3) / 1e9, "unit": "GPair/s", "frac": _frac(c["pairs"], kms, peak),
            "pipeline_frac": _frac(c["pairs"], dms, peak), "gpu_launches_per_step": nl,
            "timing": "ms: CUDA events over the device pipeline (statistics, seeds, sweep, merge, epilogue); "
                      "host_api_ms adds the host copies"}
    if have_ref:
        cnt = c["t"].size - c["m"] + 1
        e = c["m"] // 2
        pairs_ref = (cnt - e - 1) * (cnt - e) // 2
        dt = _timed(lambda: O.ref_self_join(c["t"], c["m"], threads=threads))
        line["cpu_baseline"] = cpu_line(pairs_ref / dt / 1e9, "GPair/s",
                                        "full run of the reference self_join, whose exclusion is fixed at m/2 = 125 "
                                        "(profiles.hpp:273): %d pairs in %.2f s" % (pairs_ref, dt), False)
    out["C2"] = line

    # ---- C3: learn (from the C2 series) -> join 2^20 -> top-20 discords
    c = W.c3()
    m = c["m"]
    d_q = torch.from_numpy(c["q"]).to(dev)
    rows = c["q"].size - m + 1
    d_val = torch.empty(rows, dtype=torch.float64, device=dev)
    d_idx = torch.empty(rows, dtype=torch.int64, device=dev)
    cfg = W.c3_learn_config()
    runs = []
    for it in range(4):  # the whole pipeline through the public calls, cold plan each time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        D = tsd.learn_dictionary(c["train"], cfg)
        t1 = time.perf_counter()
        plan = tsd.DictPlan(D, m)
        plan.join_device(d_q.data_ptr(), [c["q"].size], d_val.data_ptr(), d_idx.data_ptr(), stream.cuda_stream)
        disc = tsd.find_discords((d_val.data_ptr(), rows, m), D.e_max, c["top_k"])
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        plan.close()
        if it > 0:
            runs.append((t1 - t0, t2 - t1))
    learn_s, rest_s = (statistics.median(r[i] for r in runs) for i in range(2))
    # the streaming join itself on a resident dictionary (warm plan), timed like C1 / C5
    cols = sum(s.length() - m + 1 for s in D.segments)
    cells3 = rows * cols
    c3cfg = {"m": m, "segs": [s.values for s in D.segments], "starts": [s.start for s in D.segments],
             "source_length": D.source_length}
    step_ms, k_ms, nl = _plan_config(c3cfg, [c["q"]], dev, stream, flush, peak, steps=10)
    an = np.asarray(c["anomalies"])
    hits = sum(bool(np.any(np.abs(an - d.start) <= 300)) for d in disc)
    line = {"workload": "C3: learn a dictionary from the C2 series (m=200, 2048-sample contexts, sample budget "
                        "65536) -> join the 2^20-sample anomalous ECG query (seed 3) -> top-20 discords, FP64",
            "segments": len(D.segments), "stored_samples": D.stored_samples(), "cells": cells3,
            "ms": step_ms, "kernel_ms": k_ms, "value": cells3 / (step_ms * 1e-3) / 1e9, "unit": "GCell/s",
            "frac": _frac(cells3, k_ms, peak), "gpu_launches_per_step": nl,
            "learn_ms": learn_s * 1e3, "join_and_discords_ms": rest_s * 1e3,
            "pipeline_ms": (learn_s + rest_s) * 1e3, "discords_near_injected_anomalies": int(hits),
            "timing": "ms / value: CUDA events of the join step on the resident dictionary (warm plan, L2 flushed); "
                      "learn_ms and join_and_discords_ms: host wall time of the public calls, cold plan (median "
                      "of 3 after one warm run)"}
    if have_ref:
        tl = _timed(lambda: O.ref_learn_dictionary_full(c["train"], m, k=c["k"], rule=1, value=c["budget"],
                                                        threads=threads))
        w = rows if args.cpu_c3_windows <= 0 else min(rows, args.cpu_c3_windows)
        segs = [s.values for s in D.segments]
        starts = [s.start for s in D.segments]
        tj = _timed(lambda: O.ref_join_dictionary(c["q"][: w + m - 1], segs, starts, m, threads=threads))
        vals = d_val.cpu().numpy()
        td = _timed(lambda: O.ref_find_discords(vals, m, D.e_max, c["top_k"]))
        line["cpu_baseline"] = cpu_line(w * cols / tj / 1e9, "GCell/s",
                                        "reference learn_dictionary (full, %.2f s), join_dictionary on the first %d "
                                        "query windows (%.2f s), find_discords (%.3f s)" % (tl, w, tj, td), w < rows)
        line["cpu_baseline"]["pipeline_s"] = tl + tj * rows / w + td
    del d_q, d_val, d_idx
    out["C3"] = line

    # ---- C5: 4096 series x 8192 vs 64 x 1024, m = 128, one device pass
    c = W.c5()
    ms, kms, nl = _plan_config(c, list(c["series"]), dev, stream, flush, peak, steps=3)
    line = {"workload": "C5: 4096 traffic-like series x 8192 (seed 6) vs 64 segments x 1024 (seed 7), m=128, "
                        "one batched device pass, FP64", "cells": c["cells"], "ms": ms, "kernel_ms": kms,
            "value": c["cells"] / (ms * 1e-3) / 1e9, "unit": "GCell/s", "frac": _frac(c["cells"], kms, peak),
            "gpu_launches_per_step": nl}
    if have_ref:
        ns = 16
        dt = _timed(lambda: [O.ref_join_dictionary(c["series"][k], c["segs"], c["starts"], c["m"], threads=threads)
                             for k in range(ns)])
        cells_s = ns * (8192 - c["m"] + 1) * 64 * (1024 - c["m"] + 1)
        line["cpu_baseline"] = cpu_line(cells_s / dt / 1e9, "GCell/s",
                                        "reference join_dictionary looped over the first %d series (%.2f s)" % (ns, dt),
                                        True)
    out["C5"] = line
    torch.cuda.empty_cache()
    return out


def traffic_probe():
    """--traffic-probe (internal): one C4 FP64 join on device-resident inputs,
    the command measure_traffic() runs under ncu."""
    import torch
    import paper_2112_12965_b200 as tsd
    D, _ = make_dictionary()
    q = make_query(Q_SEED)
    nrows = Q_LEN - M + 1
    plan = tsd.DictPlan(D, M)
    d_q = torch.from_numpy(q).cuda()
    d_val = torch.empty(nrows, dtype=torch.float64, device="cuda")
    d_idx = torch.empty(nrows, dtype=torch.int64, device="cuda")
    plan.join_device(d_q.data_ptr(), [Q_LEN], d_val.data_ptr(), d_idx.data_ptr())
    torch.cuda.synchronize()
    plan.close()
    return 0


def measure_traffic(timeout_s=240):
    """DRAM bytes of one C4 join-kernel launch, measured in this bench run:
    ncu (dram__bytes_read.sum + dram__bytes_write.sum, the join kernel only)
    over a one-join probe of the same workload in a child process (no bench
    number is taken under the profiler). Returns (bytes, source) or (None,
    why) when ncu is unavailable or fails; TSD_BENCH_NCU=0 skips it."""
    import shutil
    import subprocess
    if os.environ.get("TSD_BENCH_NCU", "1") == "0":
        return None, "skipped (TSD_BENCH_NCU=0)"
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if not ncu:
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:k_join", "-c", "1", "--csv",
           sys.executable, os.path.abspath(__file__), "--traffic-probe"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
    except (OSError, subprocess.TimeoutExpired) as e:
        return None, "ncu failed: %s" % type(e).__name__
    import csv
    import io
    vals = {}
    lines = [l for l in r.stdout.splitlines() if l.startswith('"')]
    for row in csv.DictReader(io.StringIO("\n".join(lines))):
        name, unit = row.get("Metric Name"), row.get("Metric Unit", "")
        try:
            v = float(row.get("Metric Value", "").replace(",", ""))
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
        if name and name.startswith("dram__bytes") and scale:
            vals[name] = v * scale
    if len(vals) != 2:
        return None, "ncu returned no DRAM metrics (rc %d): %s" % (r.returncode, (r.stderr or r.stdout)[-200:])
    return sum(vals.values()), ("measured in this run: " + " ".join(cmd[:-3]).replace(sys.executable, "python")
                                + " bench.py --traffic-probe (one C4 join kernel launch)")


def algo_bytes_per_launch():
    """algorithmic bytes of one C4 join launch (SURVEY 8(d)'s
    per-unit figures): the query's row data read once (df, dg, invn, mu: 32 B
    per window), the dictionary's column data (32 B per column slot), and the
    per-group results written (16 B per row and segment group is the
    implementation's; the algorithm's output is 16 B per row)."""
    nrows = Q_LEN - M + 1
    return 32 * nrows + 32 * N_SEG * (SEG_LEN - M + 1) + 16 * nrows


def committed_traffic():
    """DRAM bytes per k_join launch from the committed ncu capture of this workload, or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_k_join_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_launch"]) if d.get("workload") == workload_config()["workload"] else None
    except (OSError, ValueError, KeyError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-windows", type=int, default=0,
                    help="query windows of C4 per reference-arm step (bounded sample); 0 = sized from the first "
                         "warm-up step: 2^15 .. 2^17 windows so that the run takes about 150 s")
    ap.add_argument("--cpu-c3-windows", type=int, default=1 << 18,
                    help="query windows of C3 timed for its CPU baseline (0 = all, the full run)")
    ap.add_argument("--skip-configs", action="store_true", help="only the C4 headline (+ fp32, self-join) lines")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per join launch from an ncu capture (reported as roofline.traffic)")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.traffic_probe:
        return traffic_probe()
    if args.warmup < 3:
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

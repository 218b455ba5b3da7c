#!/usr/bin/env python3
"""bench.py -- the hot path (the lifted FFT) timed on B200, plus the oracle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfgX] [--impl reference]

A "step" is one moa_fft_exec of the workload (every pass of the lifted FFT over
one batch of synthetic input already resident in HBM).  The headline workload
(default) is cfg5, the 1024^3 complex128 3-D FFT: BASELINE.json quotes its
metric "at 1/2/4/8 B200", i.e. on the partitioned configs, and cfg5 is the
largest of them that fits one GPU.  The same JSON line carries a sub-record per
other config (`configs`: cfg1-cfg4 at N=1; the partitioned cfg4 at N>1), each
timed the same way.  One JSON line is printed by rank 0.  For N > 1 (torchrun,
one process per GPU) cfg1-cfg3 run as independent per-rank replicas (weak
scaling); cfg4 / cfg5 are partitioned over the ranks (strong scaling).

Roofline accounting: a step's algorithmic HBM bytes are
ALG_PASSES round trips of the array (1 cfg1/cfg2, 2 cfg3/cfg4, 3 cfg5; 4 for
the partitioned cfg4, 3 for the partitioned cfg5), split evenly over the
kernel launches that complete the step; `roofline.frac` is the dominant
launch's share of those bytes over its CUDA-event time and the measured peak.
Its copy efficiency (a full round trip of the array per launch) is reported
separately as `copy_frac`.

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload on the host cores: the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FFT GFLOP/s (5n·log2n/t) and achieved HBM GB/s vs peak, at 1/2/4/8 B200"

WORKLOADS = {
    "cfg1": dict(desc="single 1D forward complex128 FFT, n=2^10, uniform, seed 0", n=1 << 10, batch=1,
                 dtype="c128", kind="1d"),
    "cfg2": dict(desc="batched 1D forward complex128 FFT, n=2^16, batch=1024 rows (1 GiB), uniform, seed 1",
                 n=1 << 16, batch=1024, dtype="c128", kind="1d"),
    "cfg3": dict(desc="single 1D forward complex128 FFT, n=2^28 (4 GiB), normal, seed 2; BASELINE.json names a "
                      "2^14 x 2^14 six-step lifting (2 HBM round trips): the plan's lifting is in `lifting`, its "
                      "extra round trips are charged in step_frac", n=1 << 28, batch=1,
                 dtype="c128", kind="1d"),
    "cfg4": dict(desc="single 1D forward complex64 FFT, n=2^30 (8 GiB), uniform, seed 3", n=1 << 30, batch=1,
                 dtype="c64", kind="1d", partitioned=True),
    "cfg5": dict(desc="3D forward complex128 FFT 1024^3 (16 GiB), normal, seed 4", shape=(1024, 1024, 1024),
                 dtype="c128", kind="3d", partitioned=True),
}
# HBM round trips (passes) of the algorithm per config
ALG_PASSES = {"cfg1": 1, "cfg2": 1, "cfg3": 2, "cfg4": 2, "cfg5": 3}
ALG_PASSES_DIST = {"cfg4": 4, "cfg5": 3}     # per GPU on N/p
ALG_EXCHANGES_DIST = {"cfg4": 3, "cfg5": 1}  # all-to-alls
HEADLINE = "cfg5"


def flops_per_step(w, ranks_units=1):
    if w["kind"] == "3d":
        N = w["shape"][0] * w["shape"][1] * w["shape"][2]
        return 5.0 * N * math.log2(N)
    return 5.0 * w["n"] * math.log2(w["n"]) * w["batch"] * ranks_units


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting", 0x10: "sync_boost"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(s)}


def host_info():
    """CPU model, logical CPUs and RAM of the host the oracle runs on."""
    model, mem = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "host_ram_gib": mem}


def oracle_sample(wname, budget_s):
    """Time the oracle (as it stands) on a bounded sample of the workload.
    -> (GFLOP/s, sample description, threads)."""
    import numpy as np

    import oracle
    import synth

    w = WORKLOADS[wname]
    thr = oracle.max_threads()
    if wname in ("cfg1", "cfg2"):
        n = w["n"]
        rows_per_chunk = 4096 if n <= 1024 else 16
        x = synth.fill(n * rows_per_chunk, synth.CONFIGS[wname]["seed"], synth.CONFIGS[wname]["dist"])
        rows, t0 = 0, time.perf_counter()
        while True:
            a = x.copy()
            oracle.fft_radix2_rows_inplace(a, n)
            rows += rows_per_chunk
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
        gf = 5.0 * n * math.log2(n) * rows / el / 1e9
        return gf, f"{rows} rows of the {wname} workload (n={n}, complex128 radix-2 oracle O1+O2), {el:.1f} s", thr
    # single huge transforms: one oracle transform of a scaled-down length of the same kind
    if w["kind"] == "3d":
        s = 256
        x = synth.fill(s ** 3, 4, synth.NORMAL).reshape(s, s, s)
        t0 = time.perf_counter()
        oracle.fft3d_inplace(x)
        el = time.perf_counter() - t0
        N = s ** 3
        return 5.0 * N * math.log2(N) / el / 1e9, f"one {s}^3 complex128 3-D oracle FFT (O5; cfg5 scaled 1/64), {el:.1f} s", thr
    n = 1 << 24
    x = synth.fill(n, synth.CONFIGS[wname]["seed"], synth.CONFIGS[wname]["dist"])
    t0 = time.perf_counter()
    oracle.fft_radix2_inplace(x)
    el = time.perf_counter() - t0
    return (5.0 * n * math.log2(n) / el / 1e9,
            f"one 2^24-point complex128 radix-2 oracle FFT ({wname} length scaled down), {el:.1f} s", thr)


def run_reference(args, w, rank):
    """The reference arm: the CPU oracle as it stands, on a bounded sample of the
    headline workload (each step one sample), rank 0 only."""
    if rank != 0:
        return 0
    import numpy as np

    wname = args.workload
    vals, secs = [], []
    sample = thr = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        gf, sample, thr = oracle_sample(wname, budget_s=1.0)
        if i >= args.warmup:
            vals.append(gf)
            secs.append(time.perf_counter() - t0)
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # each step is the bounded sample (cpu_baseline.sample), timed on the host
        "ms_per_step": round(float(np.median(secs)) * 1e3, 3),
        "ms_per_step_basis": "measured wall time of one bounded sample (see cpu_baseline.sample)",
        "ms_per_full_step_extrapolated": round(flops_per_step(w) / (v * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{wname}: {w['desc']}", "sample_of_workload": True},
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": thr, "kind": "oracle",
                         "sample": sample, **host_info()},
        "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sampled_error(wname, xh, y, w):
    """Part of the cpu_baseline leg (the one place bench.py may call oracle/):
    the GPU output at sampled bins against the O(n^2) definition evaluated by
    the oracle -- max |X_gpu[k] - X[k]| / (sqrt(n) rms(x)) (DESIGN.md reading
    R14).  The whole-vector rel-L2 at full size is the -m gpu tests' job
    (tests/test_gpu_parity.py, profiles/r2_*parity_full*)."""
    import numpy as np
    import torch

    import oracle

    rng = np.random.default_rng(99)
    if w["kind"] == "3d":
        s = w["shape"]
        ks = np.array([(0, 0, 0), (s[0] - 1, s[1] // 2, 7)] + [tuple(int(v) for v in rng.integers(0, s[0], 3))
                                                               for _ in range(4)], dtype=np.int64)
        ref = oracle.dft3_bins(xh.reshape(s), s, ks)
        flat = torch.from_numpy((ks[:, 0] * s[1] + ks[:, 1]) * s[2] + ks[:, 2]).to(y.device)
        got = y[flat].cpu().numpy().astype(np.complex128)
        N = s[0] * s[1] * s[2]
    else:
        n, b = w["n"], w["batch"]
        N = n
        nb = 8
        bins = np.concatenate([[0, 1, n - 1], rng.integers(0, n, nb - 3)]).astype(np.int64)
        rows = rng.integers(0, b, nb).astype(np.int64) if b > 1 else None
        ref = oracle.dft_bins(xh, n, bins, rows)
        flat = torch.from_numpy(bins + (rows * n if rows is not None else 0)).to(y.device)
        got = y[flat].cpu().numpy().astype(np.complex128)
    scale = math.sqrt(N) * float(np.sqrt(np.mean(np.abs(xh[: 1 << 22].astype(np.complex128)) ** 2)))
    return {"max_err_over_sqrt_n_rms": float(np.max(np.abs(got - ref)) / scale), "bins": int(len(ref)),
            "tol": 1e-11 if w["dtype"] == "c128" else 2e-5}


def run_config(wname, m, args, ctx, steps, warmup, e2e_steps, headline):
    """Time one workload; -> its record (every field of the JSON line but the
    run-level ones)."""
    import numpy as np
    import torch

    import synth

    w = WORKLOADS[wname]
    world, rank, dist, td = ctx["world"], ctx["rank"], ctx["dist"], ctx["td"]
    partitioned = dist and w.get("partitioned", False)
    t0 = time.perf_counter()
    if w["kind"] == "3d":
        plan = m.FFTPlan.plan_3d(*w["shape"], dtype=w["dtype"], ngpu=world if partitioned else 1)
    else:
        plan = m.FFTPlan(w["n"], w["batch"], w["dtype"], ngpu=world if partitioned else 1)
    plan_ms = (time.perf_counter() - t0) * 1e3
    L = plan.local_elems
    esize = 16 if w["dtype"] == "c128" else 8
    cfgsyn = synth.CONFIGS[wname]
    e0 = rank * L if partitioned else 0
    xh = synth.fill(L, cfgsyn["seed"], cfgsyn["dist"], w["dtype"], e0=e0)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    data_bytes = L * esize
    small = data_bytes * 2 < 256 << 20
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if small else None

    def barrier():
        if dist:
            td.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        plan.exec(x, y, stream)
    barrier()

    launches = plan.launches
    # the timed calls go straight to the C-ABI entry point (moa_fft_exec through
    # ctypes, pointers and stream resolved once): for the latency-bound cfg1 the
    # Python wrapper's argument checks would otherwise be part of every step
    xp, yp, sh, ph = x.data_ptr(), y.data_ptr(), stream.cuda_stream, plan.h

    def run_exec():
        m.moa_fft_exec(ph, xp, yp, sh)

    # per-launch events (moa_fft_prof_*) ride inside the timed loop, except for
    # the latency-bound small configs, where their records would be part of the
    # step: those take the per-launch times from a separate loop afterwards
    if not small:
        m.moa_fft_prof_begin(plan.h, steps)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)] if small else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx["local"]) as clk:
        barrier()
        if small:
            for i in range(steps):
                flush.fill_(i & 0xFF)                        # evict L2 between timed iterations
                ev[2 * i].record(stream)
                run_exec()
                ev[2 * i + 1].record(stream)
            barrier()
            total_ms = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps))
        else:
            start.record(stream)
            for _ in range(steps):
                run_exec()
            end.record(stream)
            barrier()
            total_ms = start.elapsed_time(end)
    if small:
        m.moa_fft_prof_begin(plan.h, steps)
        for i in range(steps):
            flush.fill_(i & 0xFF)
            run_exec()
        barrier()
    step_ms_list, nexec = m.moa_fft_prof_end(plan.h)
    ms = total_ms / steps
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        ms = float(t.item())

    units = world if (dist and not partitioned) else 1
    flops = flops_per_step(w, units)
    value = flops / (ms * 1e-3) / 1e9

    # ---- per-launch accounting
    peak, peak_src = load_peaks()
    desc = plan.describe()
    vt = "double2" if w["dtype"] == "c128" else "float2"
    launches_l = []
    xchg = []                                    # (step index, per-peer elements) of every all-to-all
    if partitioned:
        sched = m.moa_dist_describe(rank, world, w["shape"] if w["kind"] == "3d" else w["n"], w["dtype"])
        for s in sched["steps"]:
            if s[0] in ("pass", "fused"):
                launches_l.append((s[0], f"pass_kernel<{vt},{sched['passes'][s[1]]['logR']}>"))
                if s[0] == "fused":
                    xchg.append((len(launches_l) - 1, s[3], "fused into the pass's NVLink stores"))
            elif s[0] == "barrier":
                launches_l.append(("barrier", "ncclAllReduce(1)"))
            else:
                launches_l.append(("alltoall", "ncclAlltoAll"))
                xchg.append((len(launches_l) - 1, s[3], "ncclAlltoAll"))
    else:
        i = 0
        while i < len(desc):
            if desc[i]["ring"] == 2:
                launches_l.append(("pair", f"pair_kernel<{vt},{desc[i]['logR']},{desc[i + 1]['logR']}>"))
                i += 2
            else:
                dd = desc[i]
                # the TMA-store form (kernels.cu launch_t: complex128 512- / 1024-point
                # passes with contiguous loads and transposed stores)
                st_env = os.environ.get("MOA_FFT_TMA_ST")
                auto_st = vt == "double2" or os.environ.get("MOA_FFT_TMA_ST64") == "1"
                tma_st = (dd["logR"] in (9, 10) and not dd["lf_load"] and dd["lf_store"]
                          and dd.get("kind", 0) == 0 and not dd["ring"]
                          and (st_env == "1" if st_env is not None else auto_st))
                launches_l.append(("pass", f"pass_kernel{'_st' if tma_st else ''}<{vt},{dd['logR']}>"))
                i += 1
    per_step = [s / max(nexec, 1) for s in step_ms_list]
    if len(launches_l) != len(per_step):
        launches_l = [("pass", f"step {i}") for i in range(len(per_step))]
        xchg = []
    kinds = [k for k, _ in launches_l]
    pass_idx = [i for i, k in enumerate(kinds) if k in ("pass", "pair", "fused")]
    dom = max(pass_idx, key=lambda i: per_step[i])
    dom_ms = per_step[dom]
    alg_passes = ALG_PASSES_DIST[wname] if partitioned else ALG_PASSES[wname]
    step_alg_bytes = alg_passes * 2 * data_bytes         # per GPU
    launch_alg_bytes = step_alg_bytes / len(pass_idx)    # the step's bytes split over its pass launches
    achieved = launch_alg_bytes / (dom_ms * 1e-3) / 1e9
    copy_gbs = 2 * data_bytes / (dom_ms * 1e-3) / 1e9    # a full round trip of the array per launch
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        ent = tr.get(wname, {}).get(launches_l[dom][1])
        if ent is not None:
            traffic = ent if isinstance(ent, (int, float)) else ent.get("bytes")
    except Exception:
        pass
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": traffic,
        "traffic_source": "ncu --set full capture (profiles/traffic.json), per launch" if traffic else None,
        "kernel": f"{launches_l[dom][1]} (step {dom})", "kernel_ms": round(dom_ms, 4),
        "kernel_alg_bytes": int(launch_alg_bytes), "peak_source": peak_src,
        "alg_round_trips": alg_passes, "launches_completing_step": len(pass_idx),
        "copy_frac": round(copy_gbs / peak, 4), "copy_gbs": round(copy_gbs, 1),
        "step_alg_bytes": int(step_alg_bytes),
        "step_frac": round(step_alg_bytes / (ms * 1e-3) / 1e9 / peak, 4),
        "spec_peak": 8000.0, "step_frac_of_spec": round(step_alg_bytes / (ms * 1e-3) / 1e9 / 8000.0, 4),
        "per_step_ms": [round(v, 4) for v in per_step], "step_kinds": kinds,
    }
    nvlink = None
    if partitioned and xchg:
        # bytes each GPU sends per exchange = (p-1)/p * D/p; NVLink
        # 900 GB/s per direction (spec), 770 GB/s measured peer copy (B200_PROFILING.md)
        ex = []
        for si, cnt, how in xchg:
            b = (world - 1) * cnt * esize
            ex.append({"step": si, "how": how, "bytes_per_gpu": int(b), "ms": round(per_step[si], 4),
                       "GBps": round(b / (per_step[si] * 1e-3) / 1e9, 1) if how == "ncclAlltoAll" else None})
        nvl_bytes = ALG_EXCHANGES_DIST[wname] * (world - 1) * (L // world) * esize
        t_roof = step_alg_bytes / (peak * 1e9) + nvl_bytes / 770e9
        nvlink = {"exchanges": ex, "alg_nvlink_bytes_per_gpu": int(nvl_bytes), "nvlink_peak_GBps": 770.0,
                  "nvlink_peak_source": "B200_PROFILING.md measured peer copy (900 nominal)",
                  "combined_roofline_ms": round(t_roof * 1e3, 4),
                  "combined_frac": round(t_roof * 1e3 / ms, 4)}

    e2e = None
    if e2e_steps > 0:
        hin = torch.from_numpy(xh).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        plan.exec_host(hin, hout, stream)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(e2e_steps):
            plan.exec_host(hin, hout, stream)
        s1.record(stream)
        barrier()
        ems = s0.elapsed_time(s1) / e2e_steps
        if dist:
            t = torch.tensor([ems], device="cuda", dtype=torch.float64)
            td.all_reduce(t, op=td.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": round(flops / (ems * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": data_bytes, "d2h_bytes_per_step": data_bytes, "ms_per_step": round(ems, 3),
               "steps": e2e_steps}
        del hin, hout

    latency = None
    if small and not partitioned and rank == 0:
        def med(fn, reps=1000):
            ts = []
            for _ in range(reps):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                fn()
                a1.record(stream)
                a1.synchronize()
                ts.append(a0.elapsed_time(a1) * 1e3)
            return round(sorted(ts)[len(ts) // 2], 2)
        plain_us = med(run_exec)
        wrapper_us = med(lambda: plan.exec(x, y, stream))
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                plan.exec(x, y, side)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=side):
                    plan.exec(x, y, side)
            stream.wait_stream(side)
            graph_us = med(g.replay)
        except Exception as ex:  # pragma: no cover
            graph_us = f"capture failed: {ex}"
        # and with L2 flushed before each call (the timed region's condition)
        fl = []
        for i in range(200):
            flush.fill_(i & 0xFF)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            run_exec()
            a1.record(stream)
            a1.synchronize()
            fl.append(a0.elapsed_time(a1) * 1e3)
        # device-side time of one call: a sleep kernel ahead of the events keeps
        # the GPU busy while the host enqueues, so the host's submission time
        # stays outside the event pair (the flushed figure above gets the same
        # effect from its fill kernel)
        dv = []
        for i in range(200):
            torch.cuda._sleep(20000)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            run_exec()
            a1.record(stream)
            a1.synchronize()
            dv.append(a0.elapsed_time(a1) * 1e3)
        de = []
        for i in range(200):
            torch.cuda._sleep(20000)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            torch.cuda._sleep(0)
            a1.record(stream)
            a1.synchronize()
            de.append(a0.elapsed_time(a1) * 1e3)
        latency = {"device_us_warm": round(sorted(dv)[len(dv) // 2], 2),
                   "device_empty_kernel_us": round(sorted(de)[len(de) // 2], 2),
                   "plain_launch_us": plain_us, "plain_launch_l2_flushed_us": round(sorted(fl)[len(fl) // 2], 2),
                   "python_wrapper_us": wrapper_us, "cuda_graph_us": graph_us, "l2": "warm unless stated",
                   "reps": 1000, "how": "CUDA events around one moa_fft_exec C-ABI call (ctypes), median"}

    err = None
    if ctx["cpu_leg"]:
        plan.exec(x, y, stream)
        torch.cuda.synchronize()
        try:
            err = sampled_error(wname, xh, y, w)
        except Exception as ex:  # pragma: no cover
            err = {"error": str(ex)}

    rec = {
        "workload": f"{wname}: {w['desc']}", "dtype_elem": w["dtype"],
        "lifting": [d["R"] for d in desc] if w["kind"] == "1d" and not partitioned else None,
        "passes": len(desc), "plan_ms": round(plan_ms, 1),
        "l2": "L2 flushed (512 MiB write) before every timed iteration" if small else
        f"inputs larger than L2 ({data_bytes / 2**30:.2f} GiB in + out per rank)",
        "parallelism": (f"processor-lifted over {world} ranks" if partitioned else
                        (f"{world} independent replicas" if dist else "1 GPU")),
        "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 5), "value": round(value, 3),
        "unit": "GFLOP/s", "scaling": "strong" if partitioned else "weak",
        "roofline": roofline, "e2e": e2e, "launches_per_step": launches, "clocks": clk.result(),
    }
    if w["kind"] == "1d":
        rec.update(n=w["n"], batch=w["batch"])
    else:
        rec.update(shape=list(w["shape"]))
    if latency:
        rec["latency"] = latency
    if nvlink:
        rec["nvlink"] = nvlink
    if err:
        rec["sampled_parity"] = err
    plan.close()
    del x, y, xh, flush
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=HEADLINE, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub-configs", action="store_true", help="time only --workload")
    ap.add_argument("--e2e-steps", type=int, default=2)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import torch

    import paper_0803_2386_b200 as m

    torch.cuda.set_device(local)
    dist = world > 1
    td = None
    if dist:
        # NCCL's INFO init lines (communicator rank counts) stay visible to the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    subs = [] if args.no_sub_configs else (
        [c for c in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5") if c != args.workload] if not dist else
        [c for c in ("cfg4", "cfg5") if c != args.workload])
    need_dist = dist and any(WORKLOADS[c].get("partitioned", False) for c in [args.workload] + subs)
    if need_dist:
        uid = [m.moa_fft_get_unique_id() if rank == 0 else None]
        td.broadcast_object_list(uid, src=0)
        m.moa_fft_dist_init(rank, world, uid[0])
    ctx = dict(world=world, rank=rank, local=local, dist=dist, td=td,
               cpu_leg=(rank == 0 and world == 1 and not args.no_cpu_baseline))

    head = run_config(args.workload, m, args, ctx, args.steps, args.warmup, args.e2e_steps, True)
    sub = {}
    for c in subs:
        sub[c] = run_config(c, m, args, ctx, min(args.steps, 20), args.warmup, 1, False)

    cpu = None
    if ctx["cpu_leg"]:
        gf, sample, thr = oracle_sample(args.workload, budget_s=12.0)
        cpu = {"value": round(gf, 3), "unit": "GFLOP/s", "cores": thr, "kind": "oracle", "sample": sample,
               **host_info()}

    if rank == 0:
        cfg = {k: head[k] for k in ("workload", "dtype_elem", "lifting", "passes", "plan_ms", "l2", "parallelism")}
        for k in ("n", "batch", "shape", "latency", "nvlink", "sampled_parity"):
            if k in head:
                cfg[k] = head[k]
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": head["scaling"], "vs_baseline": None,
            "dtype": "f64" if w["dtype"] == "c128" else "f32", "data": "synthetic (synth/, SURVEY §8(d.4) recipe)",
            "config": cfg, "roofline": head["roofline"], "cpu_baseline": cpu, "e2e": head["e2e"],
            "gpu_launches": head["launches_per_step"] * args.steps, "clocks": head["clocks"],
            "configs": sub,
        }
        print(json.dumps(line), flush=True)
    if need_dist:
        m.moa_fft_dist_finalize()
    if dist:
        td.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

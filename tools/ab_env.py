#!/usr/bin/env python3
"""A/B timing of plan environments (ablation knobs) on the bench configs.

  ab_env.py --cases cfg3,cfg5 --variants "base:" "pf1:MOA_FFT_PF=1" "pf2:MOA_FFT_PF=2" [--reps 10]

Each variant is name:ENV=V[,ENV=V...]; the variants of one case alternate
(round-robin over --rounds) so box drift hits all of them alike.  Prints one
JSON line per (case, variant, round): total ms per exec (CUDA events over
--reps execs) and per-launch ms (the library's per-step events).
"""
import argparse
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

LAST_CLK = {}
CASES = {
    "cfg2": dict(n=1 << 16, batch=1024, dtype="c128"),
    "cfg3": dict(n=1 << 28, batch=1, dtype="c128"),
    "cfg4": dict(n=1 << 30, batch=1, dtype="c64"),
    "cfg5": dict(shape=(1024, 1024, 1024), dtype="c128"),
    "cfg5c64": dict(shape=(1024, 1024, 1024), dtype="c64"),
    "c128_2p26": dict(n=1 << 26, batch=1, dtype="c128"),
    "c64_2p28": dict(n=1 << 28, batch=1, dtype="c64"),
}


def parse_case(s):
    if s in CASES:
        return CASES[s]
    # n:batch:dtype[:lift r0.r1...]  or  shape a.b.c:dtype
    f = s.split(":")
    if "." in f[0] and f[0].count(".") == 2:
        return dict(shape=tuple(int(v) for v in f[0].split(".")), dtype=f[1])
    c = dict(n=int(f[0]), batch=int(f[1]), dtype=f[2])
    if len(f) > 3:
        c["lift"] = [int(v) for v in f[3].split(".")]
    return c


class Nvml:
    """SM clock / power samples during a timed region (median)."""

    def __init__(self):
        import threading
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(0)
            self.ok = True
        except Exception:
            pass
        self.threading = threading

    def __enter__(self):
        self.clk, self.pw, self.stop = [], [], self.threading.Event()
        if self.ok:
            def loop():
                while not self.stop.is_set():
                    try:
                        self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                        self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                    except Exception:
                        pass
                    self.stop.wait(0.002)
            self.t = self.threading.Thread(target=loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.clk:
            return {}
        c, p = sorted(self.clk), sorted(self.pw)
        return {"sm_mhz": c[len(c) // 2], "power_w": round(p[len(p) // 2], 1), "samples": len(c)}


def run(case, reps):
    if "shape" in case:
        plan = m.FFTPlan.plan_3d(*case["shape"], dtype=case["dtype"])
    else:
        plan = m.FFTPlan(case["n"], case["batch"], case["dtype"], radices=case.get("lift"))
    dt = torch.complex128 if case["dtype"] == "c128" else torch.complex64
    x = torch.randn(plan.local_elems, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        plan.exec(x, y)
    torch.cuda.synchronize()
    m.moa_fft_prof_begin(plan.h, reps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Nvml() as nv:
        e0.record()
        for _ in range(reps):
            plan.exec(x, y)
        e1.record()
        torch.cuda.synchronize()
    global LAST_CLK
    LAST_CLK = nv.summary()
    per, nex = m.moa_fft_prof_end(plan.h)
    desc = [(1 << d["logR"], d["W"], d["threads"]) for d in plan.describe()]
    plan.close()
    del x, y
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps, [round(v / max(nex, 1), 4) for v in per], desc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg3")
    ap.add_argument("--variants", nargs="+", default=["base:"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=2)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base_env = dict(os.environ)
    for cs in a.cases.split(","):
        case = parse_case(cs)
        for rnd in range(a.rounds):
            for v in a.variants:
                name, _, envs = v.partition(":")
                os.environ.clear()
                os.environ.update(base_env)
                for kv in filter(None, re.split(r",(?=[A-Z_0-9]+=)", envs)):
                    k, _, val = kv.partition("=")
                    os.environ[k] = val
                try:
                    ms, per, desc = run(case, a.reps)
                    print(json.dumps({"case": cs, "variant": name, "env": envs, "round": rnd, "ms": round(ms, 4), "clk": LAST_CLK,
                                      "per_launch_ms": per, "passes": desc}), flush=True)
                except Exception as ex:  # keep sweeping
                    print(json.dumps({"case": cs, "variant": name, "env": envs, "round": rnd, "error": str(ex)}),
                          flush=True)
    os.environ.clear()
    os.environ.update(base_env)


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Validate the planner: for n = 2^t (one transform) and each
dtype, time the planner's lifting against every other lifting into 2-4
power-of-two factors drawn from {2^5 .. 2^11} (last pass up to 2^12), CUDA
events over --reps execs, and report which wins.
  planner_sweep.py [tmin tmax] [--reps R]"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402


def liftings(t):
    out = set()
    for k in (2, 3, 4):
        for f in itertools.product(range(5, 13), repeat=k):
            if sum(f) == t and all(x <= 11 for x in f[:-1]):
                out.add(f)
    return sorted(out)


def timeit(plan, x, y, reps):
    for _ in range(2):
        plan.exec(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.exec(x, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ap = argparse.ArgumentParser()
ap.add_argument("tmin", type=int, nargs="?", default=20)
ap.add_argument("tmax", type=int, nargs="?", default=28)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dtypes", default="c128,c64")
ap.add_argument("--total", type=int, default=0, help="batched: rows = 2^total / n (0: one transform)")
a = ap.parse_args()
torch.cuda.set_device(0)
for dt in a.dtypes.split(","):
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    for t in range(a.tmin, a.tmax + 1):
        n = 1 << t
        batch = (1 << a.total) // n if a.total else 1
        x = torch.randn(n * batch, dtype=tdt, device="cuda")
        y = torch.empty_like(x)
        planned = m.moa_plan_radices(n, batch, dt)
        res = []
        for f in liftings(t):
            rad = [1 << v for v in f]
            try:
                p = m.FFTPlan(n, batch, dt, radices=rad)
                res.append((timeit(p, x, y, a.reps), rad))
                p.close()
            except Exception:
                pass
        res.sort()
        tp = next((ms for ms, r in res if r == planned), None)
        print(json.dumps({"dtype": dt, "t": t, "batch": batch, "planned": planned, "planned_ms": tp and round(tp, 4),
                          "best": res[0][1], "best_ms": round(res[0][0], 4),
                          "planned_rank": next((i for i, (ms, r) in enumerate(res) if r == planned), None),
                          "candidates": len(res), "top5": [(round(ms, 4), r) for ms, r in res[:5]]}), flush=True)
        del x, y
        torch.cuda.empty_cache()

#!/usr/bin/env python3
"""Run one plan a few times (for ncu captures of individual passes).

  prof_case.py --n 268435456 --dtype c128 [--batch B] [--lift 512,512,1024] [--reps 3]
  prof_case.py --shape 512,512,512 --dtype c128
Prints per-exec ms (CUDA events) and the plan's launches per exec.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--shape", default="")
ap.add_argument("--dtype", default="c128")
ap.add_argument("--lift", default="")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
torch.cuda.set_device(0)
if a.shape:
    s = [int(v) for v in a.shape.split(",")]
    plan = m.FFTPlan.plan_3d(*s, dtype=a.dtype)
else:
    rad = [int(v) for v in a.lift.split(",")] if a.lift else None
    plan = m.FFTPlan(a.n, a.batch, a.dtype, radices=rad)
dt = torch.complex128 if a.dtype == "c128" else torch.complex64
x = torch.randn(plan.local_elems, dtype=dt, device="cuda")
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps):
    if i == a.reps - 1:
        m.moa_fft_prof_begin(plan.h, 1)
    e0.record()
    plan.exec(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(f"exec {i}: {e0.elapsed_time(e1):.3f} ms, launches/exec {plan.launches}", flush=True)
per, nex = m.moa_fft_prof_end(plan.h)
print("per-launch ms:", [round(v / max(nex, 1), 3) for v in per])
print([(d["logR"], d["W"], d["threads"], d["smem_bytes"]) for d in plan.describe()])
plan.close()  # prints MOA_FFT_STATS ring statistics, if enabled

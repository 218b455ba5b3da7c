#!/usr/bin/env python3
"""Energy split of a plan's passes: the full passes (moa_fft_exec) against the
same descriptors as pure movements (moa_pass_move), each timed with CUDA
events over --reps execs while NVML samples SM clock and board power.
  power_split.py cfg5 [--reps 30]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402
from tools.ab_env import Nvml, parse_case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("case")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--seconds", type=float, default=3.0, help="run each leg this long; NVML samples its second half")
a = ap.parse_args()
torch.cuda.set_device(0)
case = parse_case(a.case)
plan = (m.FFTPlan.plan_3d(*case["shape"], dtype=case["dtype"]) if "shape" in case
        else m.FFTPlan(case["n"], case["batch"], case["dtype"], radices=case.get("lift")))
dt = torch.complex128 if case["dtype"] == "c128" else torch.complex64
x = torch.randn(plan.local_elems, dtype=dt, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream()
desc = plan.describe()


def timed(fn, label):
    import time
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    one = max(time.time() - t0, 1e-4)
    reps = max(a.reps, int(a.seconds / 2 / one))
    for _ in range(reps):                      # first half: reach the power / thermal steady state
        fn()
    torch.cuda.synchronize()
    with Nvml() as nv:
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    c = nv.summary()
    print(json.dumps({"case": a.case, "what": label, "ms": round(ms, 4), **c,
                      "mJ": round(ms * c.get("power_w", 0), 1)}), flush=True)


timed(lambda: plan.exec(x, y), "exec (all passes)")
timed(lambda: [m.moa_pass_move(d, case["dtype"], x.data_ptr(), y.data_ptr(), s.cuda_stream) for d in desc],
      "movement only (same descriptors, DFT and weights off)")
timed(lambda: y.copy_(x), "torch copy_ of the array (x3 = passes)")

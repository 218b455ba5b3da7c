#!/usr/bin/env python3
"""Split a pass's time into access pattern and arithmetic: each descriptor of
a plan timed as the full pass (moa_fft_exec per-pass events) and as a pure
movement with the same ONF maps (moa_pass_move: DFT and weights off).
  move_vs_pass.py n batch dtype  |  move_vs_pass.py 3d n0 n1 n2 dtype"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

if sys.argv[1] == "3d":
    shape = tuple(int(v) for v in sys.argv[2:5])
    dt = sys.argv[5]
    n, B = shape[0] * shape[1] * shape[2], 1
    plan = m.FFTPlan.plan_3d(*shape, dtype=dt)
else:
    n, B, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    plan = m.FFTPlan(n, B, dt)
tdt = torch.complex128 if dt == "c128" else torch.complex64
x = torch.randn(n * B, dtype=tdt, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream()
for _ in range(3):
    plan.exec(x, y)
reps = 10
m.moa_fft_prof_begin(plan.h, reps)
for _ in range(reps):
    plan.exec(x, y)
torch.cuda.synchronize()
per, nx = m.moa_fft_prof_end(plan.h)
per = [v / max(nx, 1) for v in per]
for i, d in enumerate(plan.describe()):
    for _ in range(3):
        m.moa_pass_move(d, dt, x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        m.moa_pass_move(d, dt, x.data_ptr(), y.data_ptr(), s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    mv = e0.elapsed_time(e1) / reps
    print(json.dumps({"n": n, "batch": B, "dtype": dt, "pass": i, "R": 1 << d["logR"], "lf_load": d["lf_load"],
                      "lf_store": d["lf_store"], "twN": d["twN"], "pass_ms": round(per[i], 4),
                      "move_ms": round(mv, 4)}), flush=True)

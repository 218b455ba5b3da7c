#!/usr/bin/env python3
"""Time the processor-level lifting on ONE GPU through the loopback backend of
the product step loop (dist_exec): all p virtual ranks' kernels on this
device, exchanges as device copies or fused into the passes' stores.
HBM-only: it measures the per-rank kernels and chunk maps at full size, not
NVLink.  Prints one JSON line with the exec time and the per-step times of the
schedule (each step summed over the p virtual ranks), from which the per-GPU
pass time of a real p-GPU run is the pass time / p.
  loopback_timing.py N p dtype            (1-D, cfg4-style)
  loopback_timing.py 3d n0 n1 n2 p dtype  (3-D slab, cfg5-style)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

if sys.argv[1] == "3d":
    shape = tuple(int(v) for v in sys.argv[2:5])
    p, dt = int(sys.argv[5]), sys.argv[6]
    N = shape[0] * shape[1] * shape[2]
else:
    shape = None
    N, p, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
torch.cuda.set_device(0)
tdt = torch.complex128 if dt == "c128" else torch.complex64
plans = []
for r in range(p):
    m.moa_fft_dist_loopback(r, p)
    plans.append(m.FFTPlan.plan_3d(*shape, dtype=dt, ngpu=p) if shape else m.FFTPlan(N, 1, dt, ngpu=p))
ins = [torch.randn(N // p, dtype=tdt, device="cuda") for _ in range(p)]
outs = [torch.empty_like(x) for x in ins]
s = torch.cuda.current_stream()
args = ([pl.h for pl in plans], [x.data_ptr() for x in ins], [o.data_ptr() for o in outs], s.cuda_stream)
for _ in range(2):
    m.moa_fft_exec_loopback(*args)
reps = 5
m.moa_fft_prof_begin(plans[0].h, reps)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    m.moa_fft_exec_loopback(*args)
e1.record()
torch.cuda.synchronize()
per, nx = m.moa_fft_prof_end(plans[0].h)
sched = m.moa_dist_describe(0, p, shape if shape else N, dt)
print(json.dumps({"N": N, "shape": shape, "p": p, "dtype": dt, "peer": os.environ.get("MOA_FFT_PEER", "1"),
                  "exec_ms_all_ranks": round(e0.elapsed_time(e1) / reps, 3),
                  "steps": [s[0] for s in sched["steps"]],
                  "step_ms_all_ranks": [round(v / max(nx, 1), 3) for v in per]}), flush=True)

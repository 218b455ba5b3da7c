#!/usr/bin/env python3
"""Time the processor-level lifting on ONE GPU through the loopback executor
(all p virtual ranks' kernels on this device; exchanges as device copies, or
fused into the passes' stores).  HBM-only: shows the traffic the fused
exchange saves, not NVLink behaviour.
  loopback_timing.py N p dtype
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

N, p, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
torch.cuda.set_device(0)
tdt = torch.complex128 if dt == "c128" else torch.complex64
plans = []
for r in range(p):
    m.moa_fft_dist_loopback(r, p)
    plans.append(m.FFTPlan(N, 1, dt, ngpu=p))
ins = [torch.randn(N // p, dtype=tdt, device="cuda") for _ in range(p)]
outs = [torch.empty_like(x) for x in ins]
s = torch.cuda.current_stream()
args = ([pl.h for pl in plans], [x.data_ptr() for x in ins], [o.data_ptr() for o in outs], s.cuda_stream)
for _ in range(2):
    m.moa_fft_exec_loopback(*args)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    m.moa_fft_exec_loopback(*args)
e1.record()
torch.cuda.synchronize()
sched = m.moa_dist_describe(0, p, N, dt)
print(f"N={N} p={p} {dt} peer={os.environ.get('MOA_FFT_PEER', '1')}: {e0.elapsed_time(e1) / 5:.3f} ms per exec "
      f"(all {p} virtual ranks on one GPU); steps {[st[0] for st in sched['steps']]}")

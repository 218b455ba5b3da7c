#!/usr/bin/env python3
"""Event-to-event floor of one kernel launch on this box (what a 1-line FFT
cannot beat): torch.cuda._sleep(0) (an empty kernel) and a 16-byte copy,
medians over 2000 launches, with and without CUDA graphs."""
import json
import torch

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
x = torch.zeros(2, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)


def med(fn, reps=2000):
    ts = []
    for _ in range(reps):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(s)
        fn()
        a1.record(s)
        a1.synchronize()
        ts.append(a0.elapsed_time(a1) * 1e3)
    return round(sorted(ts)[len(ts) // 2], 2)


for _ in range(100):
    torch.cuda._sleep(0)
out = {"empty_kernel_us": med(lambda: torch.cuda._sleep(0)), "copy_16B_us": med(lambda: y.copy_(x)),
       "nothing_us": med(lambda: None)}
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    torch.cuda._sleep(0)
out["empty_kernel_graph_us"] = med(g.replay)
print(json.dumps(out))

#!/usr/bin/env python3
"""Host<->device copy ceilings for the e2e number: pinned H2D alone, D2H
alone, and both at once on two streams (1 GiB each), CUDA events."""
import json

import torch

nb = 1 << 30
h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
d_a = torch.empty(nb, dtype=torch.uint8, device="cuda")
d_b = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    for s in (s1, s2):
        e = torch.cuda.Event()
        e.record(s)
        torch.cuda.current_stream().wait_event(e)


h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
bi = timed(both)
print(json.dumps({"h2d_GBps": round(nb / h2d / 1e6, 1), "d2h_GBps": round(nb / d2h / 1e6, 1),
                  "bidirectional_GBps_total": round(2 * nb / bi / 1e6, 1)}))

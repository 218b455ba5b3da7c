#!/usr/bin/env python3
"""Prototype measurement for an L2-level lifting of batched two-pass plans
(cfg2): run the 1024 rows as chunks of C rows, each chunk a full two-pass
sub-plan whose scratch (C rows) can stay L2-resident, with S plans / streams
round-robin so consecutive chunks overlap.  No cache hints: shows launch and
overlap costs and how much of the intermediate's HBM traffic L2 absorbs.
  chunk_proto.py [n] [batch] [dtype]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dt = sys.argv[3] if len(sys.argv) > 3 else "c128"
torch.cuda.set_device(0)
tdt = torch.complex128 if dt == "c128" else torch.complex64
x = torch.randn(B, n, dtype=tdt, device="cuda")
y = torch.empty_like(x)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


full = m.FFTPlan(n, B, dt)
print(f"full plan: {timeit(lambda: full.exec(x, y)):.3f} ms", flush=True)
ref = full.exec(x, y).clone()
for C in (8, 16, 32, 64, 128):
    for S in (1, 2, 3):
        plans = [m.FFTPlan(n, C, dt) for _ in range(S)]
        streams = [torch.cuda.Stream() for _ in range(S)]

        def run():
            ev = torch.cuda.Event()
            ev.record(main)
            for s in streams:
                s.wait_event(ev)
            for c in range(B // C):
                k = c % S
                with torch.cuda.stream(streams[k]):
                    plans[k].exec(x[c * C:(c + 1) * C].reshape(-1), y[c * C:(c + 1) * C].reshape(-1), stream=streams[k])
            for s in streams:
                e = torch.cuda.Event()
                e.record(s)
                main.wait_event(e)
        ms = timeit(run)
        ok = torch.allclose(y, ref)
        print(f"chunks of {C} rows ({C * n * x.element_size() >> 20} MiB), {S} streams: {ms:.3f} ms  match={ok}",
              flush=True)

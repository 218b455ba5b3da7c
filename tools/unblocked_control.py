#!/usr/bin/env python3
"""The paper's lifted-vs-unblocked experiment (PAPER.md Ch.3 results,
P:3081-3172: "c >= n disables blocking", same code) reproduced on B200.

For n = 2^t (complex128, one transform, inputs resident in HBM) time
  * the planner's lifting (each pass one HBM round trip of <= 2^8-point blocks),
  * the unblocked control: the all-radix-2 lifting, one global radix-2 stage
    per pass (t passes) -- the Van Loan loop with no blocking,
  * the hypercube form (MOA_FFT_HYPERCUBE): the same t radix-2 stages with the
    Ch.5 stage transposes t_j done physically, one loop over (i, i + n/2) at
    every stage -- the paper's "simpler control structure" conjecture
    (P:5880-5887), which it never measured,
with CUDA events (median of reps, L2 flushed before each rep), and print one
JSON line per n.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402


def time_plan(plan, x, y, reps=5):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 1):
        flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.exec(x, y)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    torch.cuda.set_device(0)
    tmin, tmax = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (12, 26)))
    for t in range(tmin, tmax + 1):
        n = 1 << t
        x = torch.randn(n, dtype=torch.complex128, device="cuda")
        y = torch.empty_like(x)
        lifted = m.FFTPlan(n, 1, "c128")
        ms_l = time_plan(lifted, x, y)
        rad_l = [1 << d["logR"] for d in lifted.describe()]
        lifted.close()
        unb = m.FFTPlan(n, 1, "c128", unblocked=True)
        ms_u = time_plan(unb, x, y)
        unb.close()
        hyp = m.FFTPlan(n, 1, "c128", hypercube=True)
        ms_h = time_plan(hyp, x, y)
        hyp.close()
        gf = lambda ms: 5.0 * n * t / (ms * 1e-3) / 1e9
        print(json.dumps({"n": n, "lifted_radices": rad_l, "lifted_ms": round(ms_l, 4), "lifted_gflops": round(gf(ms_l), 1),
                          "unblocked_passes": t, "unblocked_ms": round(ms_u, 4),
                          "unblocked_gflops": round(gf(ms_u), 1), "speedup": round(ms_u / ms_l, 2),
                          "hypercube_ms": round(ms_h, 4), "hypercube_gflops": round(gf(ms_h), 1),
                          "hypercube_vs_unblocked": round(ms_u / ms_h, 3)}), flush=True)


if __name__ == "__main__":
    main()

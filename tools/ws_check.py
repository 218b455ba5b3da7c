#!/usr/bin/env python3
"""The asynchronously fed (TMA) pass kernel against the plain one: same plan,
MOA_FFT_WS=1 vs 0, outputs compared bit for bit (the arithmetic is the same),
then per-pass timing of both.  ws_check.py [case ...] (cases as tools/ab_env.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402
from tools.ab_env import parse_case  # noqa: E402


def mk(case):
    if "shape" in case:
        return m.FFTPlan.plan_3d(*case["shape"], dtype=case["dtype"])
    return m.FFTPlan(case["n"], case["batch"], case["dtype"], radices=case.get("lift"))


def main():
    env = "MOA_FFT_WS"
    args = sys.argv[1:]
    if args and args[0].startswith("--env="):
        env = args[0][6:]
        args = args[1:]
    cases = args or ["1048576:4:c128:512.512.4", "1048576:2:c128:1024.1024"]
    torch.cuda.set_device(0)
    for cs in cases:
        case = parse_case(cs)
        dt = torch.complex128 if case["dtype"] == "c128" else torch.complex64
        outs, times = {}, {}
        for ws in ("0", "1"):
            os.environ[env] = ws
            plan = mk(case)
            g = torch.Generator(device="cuda").manual_seed(5)
            x = torch.randn(plan.local_elems, dtype=dt, device="cuda", generator=g)
            y = torch.empty_like(x)
            for _ in range(2):
                plan.exec(x, y)
            torch.cuda.synchronize()
            outs[ws] = y.clone()
            m.moa_fft_prof_begin(plan.h, 5)
            for _ in range(5):
                plan.exec(x, y)
            torch.cuda.synchronize()
            per, nx = m.moa_fft_prof_end(plan.h)
            times[ws] = [round(v / nx, 4) for v in per]
            plan.close()
            del x, y
        same = bool(torch.equal(outs["0"], outs["1"]))
        diff = float((outs["0"] - outs["1"]).abs().max().item())
        rel = float(((outs["0"] - outs["1"]).abs().pow(2).sum() / outs["0"].abs().pow(2).sum()).sqrt().item())
        print(json.dumps({"case": cs, "bitexact": same, "maxdiff": diff, "rel_l2_vs_plain": rel, "env": env, "plain_ms": times["0"], "ws_ms": times["1"]}),
              flush=True)
        del outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Ablation: shared-memory row stride of the density-matrix gate kernel
(MOA_QG_TP_OFF = TP - TC), one gate shape per line, CUDA events, median of 10."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import paper_0803_2386_b200 as m
    n = 14
    for dt in (torch.complex128, torch.complex64):
        N = 1 << n
        rho = torch.randn(N, N, dtype=dt, device="cuda")
        for bits in ([3, 9], [0, 1], [0, 13], [0, 1, 2], [2, 7, 13]):
            q = len(bits)
            U, _ = np.linalg.qr(np.random.default_rng(q).standard_normal((1 << q, 1 << q)) + 0j)
            for _ in range(3):
                m.moa_qgate_apply(rho, n, bits, U)
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                m.moa_qgate_apply(rho, n, bits, U)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            print(json.dumps({"tp_off": os.environ.get("MOA_QG_TP_OFF", "model"), "dtype": str(dt).split(".")[1],
                              "gated_bits": bits, "ms": round(sorted(ts)[5], 4)}), flush=True)
    sys.exit(0)
for off in [None, "0", "1", "2", "4", "8"]:
    env = dict(os.environ)
    if off is not None:
        env["MOA_QG_TP_OFF"] = off
    subprocess.run([sys.executable, __file__, "--child"], env=env, check=True)

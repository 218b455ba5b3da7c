#!/usr/bin/env python3
"""Throughput of the Ch.6 density-matrix gate: one moa_qgate_apply on a
2^n x 2^n complex128 matrix (in place: one HBM round trip), CUDA events,
median of 10; reported as GB/s of algorithmic traffic (2 x matrix bytes) and
as a fraction of MEASURED_PEAKS.json hbm_gbs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0803_2386_b200 as m  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
for dt in (torch.complex128, torch.complex64):
    N = 1 << n
    rho = torch.randn(N, N, dtype=dt, device="cuda")
    nbytes = rho.numel() * rho.element_size()
    for bits in ([0], [n - 1], [0, 1], [3, 9], [0, n - 1], [0, 1, 2], [2, 7, n - 1]):
        q = len(bits)
        rng = np.random.default_rng(q)
        U, _ = np.linalg.qr(rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q)))
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
        ms = sorted(ts)[5]
        gbs = 2 * nbytes / (ms * 1e-3) / 1e9
        # arithmetic: 2 * 2^q complex multiply-adds (4 FMAs = 8 flops) per element (U B U^dagger)
        tflops = N * N * 2 * (1 << q) * 8 / (ms * 1e-3) / 1e12
        print(json.dumps({"n": n, "dtype": str(dt).split(".")[1], "gated_bits": bits, "ms": round(ms, 4),
                          "GBps": round(gbs, 1), "frac_of_measured_hbm": round(gbs / peak, 3),
                          "TFLOPs": round(tflops, 2)}), flush=True)

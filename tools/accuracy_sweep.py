#!/usr/bin/env python3
"""rel-L2 error of the GPU path against the oracle (O2 radix-2, fp64) over
sizes and liftings -- the margins behind the 1e-11 / 2e-5 tolerances."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_0803_2386_b200 as m  # noqa: E402

for dt in ("c128", "c64"):
    for t in (4, 8, 10, 12, 13, 14, 15, 16, 18, 20, 22, 24):
        n = 1 << t
        batch = max(1, (1 << 20) // n)
        x = synth.fill(n * batch, t, synth.UNIFORM, dt)
        plan = m.FFTPlan(n, batch, dt)
        y = plan.exec(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.complex128)
        ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
        err = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
        print(json.dumps({"dtype": dt, "n": n, "batch": batch, "lifting": [1 << d["logR"] for d in plan.describe()],
                          "cluster_pair": [d["ring"] for d in plan.describe()] == [3, 4],
                          "rel_l2": float(f"{err:.3e}")}), flush=True)

#!/usr/bin/env python3
"""Small runs of every kernel kind, for compute-sanitizer (memcheck / racecheck /
synccheck): one-pass, lifted passes (c128 / c64, in-place and not), the 3-D
layouts, the L2-ring pairs, the unblocked control, plan flags, and the
processor-level lifting through the loopback executor (fused and copy
exchanges).  Exits non-zero on a parity failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_0803_2386_b200 as m  # noqa: E402
import synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def one(n, batch, dtype, env=None, **kw):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        x = synth.fill(n * batch, 5, synth.UNIFORM, dtype)
        plan = m.FFTPlan(n, batch, dtype, **kw)
        y = plan.exec(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.complex128)
        sign = +1 if kw.get("inverse") else -1
        ref = oracle.fft_radix2_rows_sign(x.astype(np.complex128), n, sign)
        if kw.get("normalize"):
            ref /= n
        if kw.get("lifted_order"):
            y = y.reshape(batch, n)[:, plan.output_index()].reshape(-1)
        err = rel(y, ref)
        plan.close()
        return err
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def three(shape, dtype, rot):
    os.environ["MOA_FFT_3D_ROT"] = rot
    x = synth.fill(int(np.prod(shape)), 6, synth.NORMAL, dtype)
    plan = m.FFTPlan.plan_3d(*shape, dtype=dtype)
    y = plan.exec(torch.from_numpy(x).cuda()).cpu().numpy().reshape(shape).astype(np.complex128)
    plan.close()
    del os.environ["MOA_FFT_3D_ROT"]
    return rel(y, oracle.fft3d(x.astype(np.complex128).reshape(shape)))


def dist(N, p, peer):
    os.environ["MOA_FFT_PEER"] = peer
    x = synth.fill(N, 3, synth.UNIFORM)
    plans = []
    for r in range(p):
        m.moa_fft_dist_loopback(r, p)
        plans.append(m.FFTPlan(N, 1, "c128", ngpu=p))
    ins = [torch.from_numpy(s.copy()).cuda() for s in np.split(x, p)]
    outs = [torch.empty_like(s) for s in ins]
    m.moa_fft_exec_loopback([q.h for q in plans], [s.data_ptr() for s in ins], [o.data_ptr() for o in outs],
                            torch.cuda.current_stream().cuda_stream)
    y = np.concatenate([o.cpu().numpy() for o in outs])
    for q in plans:
        q.close()
    del os.environ["MOA_FFT_PEER"]
    return rel(y, oracle.fft_radix2(x))


torch.cuda.set_device(0)
cases = [
    ("1-pass c128", lambda: one(1 << 10, 2, "c128")),
    ("2-pass c128", lambda: one(1 << 14, 2, "c128")),
    ("2-pass c64", lambda: one(1 << 15, 2, "c64")),
    ("4-pass c128", lambda: one(1 << 16, 1, "c128", radices=[16, 16, 16, 16])),
    ("pair c128", lambda: one(1 << 12, 64, "c128", env={"MOA_FFT_FUSE": "1"})),
    ("lift4 pairs c64", lambda: one(1 << 20, 1, "c64", env={"MOA_FFT_LIFT4": "1"}, radices=[32, 32, 32, 32])),
    ("unblocked", lambda: one(1 << 12, 2, "c128", unblocked=True)),
    ("inverse+norm", lambda: one(1 << 14, 2, "c128", inverse=True, normalize=True)),
    ("lifted order", lambda: one(1 << 14, 2, "c128", lifted_order=True)),
    ("3-D classic", lambda: three((16, 32, 64), "c128", "0")),
    ("3-D rot", lambda: three((16, 32, 64), "c128", "2")),
    ("3-D c64", lambda: three((32, 16, 64), "c64", "0")),
    ("small kernel c128", lambda: one(1 << 10, 3, "c128")),
    ("small kernel c64 odd", lambda: one(1 << 11, 2, "c64")),
    ("TMA-fed line-fast", lambda: one(1 << 18, 2, "c128", env={"MOA_FFT_WS": "1"}, radices=[512, 512])),
    ("TMA-fed contiguous", lambda: one(1 << 20, 1, "c128", env={"MOA_FFT_WS": "1"}, radices=[1024, 1024])),
    ("pair radix-32 c128", lambda: one(1 << 19, 2, "c128", env={"MOA_FFT_PAIR": "1"}, radices=[512, 1024])),
    ("FP32x2 radix-32 c64", lambda: one(1 << 20, 1, "c64", radices=[1024, 1024])),
    ("hypercube", lambda: one(1 << 12, 2, "c128", hypercube=True)),
    ("dist fused p4", lambda: dist(1 << 14, 4, "1")),
    ("dist nccl-style p4", lambda: dist(1 << 14, 4, "0")),
]
bad = 0
for name, f in cases:
    err = f()
    tol = 2e-5 if "c64" in name else 1e-11
    ok = err <= tol
    bad += not ok
    print(f"{name:22s} rel-L2 {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
torch.cuda.synchronize()
sys.exit(1 if bad else 0)

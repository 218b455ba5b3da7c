"""Out-of-bounds write detection without compute-sanitizer (closed on this
pool): every kind of plan runs on buffers carved from the middle of larger
allocations whose guard regions hold a canary pattern; after the exec the
guards must be bit-identical and the input untouched (out-of-place)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
GUARD = 4096  # complex elements on each side


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def m(torch_cuda):
    import paper_0803_2386_b200 as mod
    return mod


def guarded(torch, data, dtype):
    full = torch.empty(data.size + 2 * GUARD, dtype=dtype, device="cuda")
    canary = torch.full((GUARD,), complex(-7.25e300 if dtype == torch.complex128 else -7.25e30, 1.5),
                        dtype=dtype, device="cuda")
    full[:GUARD] = canary
    full[-GUARD:] = canary
    full[GUARD:-GUARD] = torch.from_numpy(data).cuda()
    return full, canary


@pytest.mark.parametrize("case", [
    dict(n=1 << 10, batch=3), dict(n=1 << 14, batch=2), dict(n=1 << 16, batch=2, dtype="c64"),
    dict(n=1 << 20, batch=1), dict(n=1 << 12, batch=40, env={"MOA_FFT_FUSE": "1"}),
    dict(n=1 << 14, batch=2, kw={"lifted_order": True}), dict(n=1 << 12, batch=2, kw={"unblocked": True}),
    dict(n=1 << 13, batch=2, kw={"inverse": True, "normalize": True}),
    dict(shape=(16, 32, 64)), dict(shape=(32, 16, 8), dtype="c64"), dict(shape=(8, 8, 8), env={"MOA_FFT_3D_ROT": "0"}),
    # the cluster pair: 8-CTA (default) and 16-CTA (forced) clusters
    dict(n=1 << 14, batch=3), dict(n=1 << 16, batch=3, env={"MOA_FFT_CLUSTER": "1"}),
    dict(n=1 << 16, batch=2, dtype="c64", env={"MOA_FFT_CLUSTER": "1"}),
])
def test_no_out_of_bounds_writes(m, torch_cuda, monkeypatch, case):
    torch = torch_cuda
    for k, v in case.get("env", {}).items():
        monkeypatch.setenv(k, v)
    dt = case.get("dtype", "c128")
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    if "shape" in case:
        plan = m.FFTPlan.plan_3d(*case["shape"], dtype=dt)
    else:
        plan = m.FFTPlan(case["n"], case["batch"], dt, **case.get("kw", {}))
    x = synth.fill(plan.local_elems, 17, synth.UNIFORM, dt)
    fin, canary = guarded(torch, x, tdt)
    fout, _ = guarded(torch, np.zeros_like(x), tdt)
    plan.exec(fin[GUARD:-GUARD], fout[GUARD:-GUARD])
    torch.cuda.synchronize()
    for buf in (fin, fout):
        assert torch.equal(buf[:GUARD], canary) and torch.equal(buf[-GUARD:], canary)
    assert np.array_equal(fin[GUARD:-GUARD].cpu().numpy(), x)          # the input is not modified
    assert np.isfinite(fout[GUARD:-GUARD].cpu().numpy()).all()

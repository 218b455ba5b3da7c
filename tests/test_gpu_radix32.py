"""GPU parity of the radix-32 steps (complex128 1024-point lines: 32 points per
thread, one shared-memory exchange, w_32 register network, pad-per-32 shared
layout) in every position a 1024-point pass takes: a single pass, the strided
first / middle pass of a lifting (line-coalesced tiles), the contiguous last
pass (transposed store), each 3-D axis in every layout, the inverse / lifted
variants and an in-place exec -- against the oracle."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


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


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("radices,batch", [([1024], 7), ([1024, 64], 3), ([64, 1024], 2), ([1024, 1024], 1),
                                           ([16, 1024, 8], 2), ([1024, 32, 32], 1)])
def test_1024_point_passes(m, torch_cuda, radices, batch):
    torch = torch_cuda
    n = int(np.prod(radices))
    x = synth.fill(n * batch, 320 + len(radices), synth.NORMAL)
    plan = m.FFTPlan(n, batch, "c128", radices=radices)
    assert any(d["logR"] == 10 and d["threads"] == d["W"] * 32 for d in plan.describe())
    y = plan.exec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel(y, oracle.fft_radix2_rows(x, n)) <= 1e-11


@pytest.mark.parametrize("shape", [(1024, 4, 8), (4, 1024, 8), (8, 4, 1024), (32, 1024, 32)])
@pytest.mark.parametrize("rot", ["0", "1", "2"])
def test_3d_1024_axes(m, torch_cuda, monkeypatch, shape, rot):
    torch = torch_cuda
    monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
    x = synth.fill(int(np.prod(shape)), 321, synth.UNIFORM).reshape(shape)
    plan = m.FFTPlan.plan_3d(*shape, dtype="c128")
    y = plan.exec(torch.from_numpy(x.reshape(-1)).cuda()).cpu().numpy().reshape(shape)
    assert rel(y, oracle.fft3d_sign(x, -1)) <= 1e-11


def test_inverse_lifted_inplace(m, torch_cuda, monkeypatch):
    torch = torch_cuda
    n, batch = 1 << 20, 2
    monkeypatch.setenv("MOA_FFT_LIFT", "1024,1024")        # the run-time lifting override (flags allowed)
    x = synth.fill(n * batch, 322, synth.UNIFORM)
    inv = m.FFTPlan(n, batch, "c128", inverse=True, normalize=True)
    assert [1 << d["logR"] for d in inv.describe()] == [1024, 1024]
    xt = torch.from_numpy(x).cuda()
    inv.exec(xt, xt)                                        # in place
    assert rel(xt.cpu().numpy(), oracle.fft_radix2_rows_sign(x, n, +1) / n) <= 1e-11
    lifted = m.FFTPlan(n, 1, "c128", lifted_order=True)
    y = lifted.exec(torch.from_numpy(x[:n].copy()).cuda()).cpu().numpy()
    pos = lifted.output_index()
    assert rel(y[pos], oracle.fft_radix2_rows(x[:n], n)) <= 1e-11

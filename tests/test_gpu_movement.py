"""Bit-exact index movement of the kernels (BASELINE.json: "the
lifting/index maps must be bit-exact against the oracle's index permutation").

Every pass descriptor of a set of plans is executed on the GPU as a pure data
movement (moa_pass_move: the DFT and the twiddles switched off) on an integer
payload x[i] = i (exact in both complex64 and complex128), and the result must
equal, element for element, the movement the descriptor's ONF prescribes --
out[store(line, k)] = in[load(line, k)] -- evaluated on the host by the
test-side ONF interpreter (tests/onf.py), which is itself checked bit-exactly
against the oracle's MoA-materialised maps in tests/test_abi_cpu.py."""
import numpy as np
import pytest

from onf import enumerate_pass

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


def descriptors(m, monkeypatch):
    out = []
    for n, batch, dt, rad in [(1 << 10, 3, "c128", None), (1 << 16, 2, "c128", None), (1 << 16, 2, "c64", None),
                              (1 << 20, 1, "c64", None), (1 << 20, 1, "c128", [128, 128, 64]),
                              (1 << 18, 1, "c128", [8, 32, 1024]), (1 << 12, 5, "c128", [2, 2048]),
                              (1 << 21, 1, "c64", [1024, 2048])]:
        for d in m.moa_psi_describe(n, batch, dt, rad):
            out.append((f"1d n={n} b={batch} {dt} R={d['R']}", d, dt, n * batch))
    for rot in ("0", "2"):
        monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
        for shape, dt in [((16, 32, 64), "c128"), ((64, 8, 1024), "c128"), ((32, 16, 1024), "c64")]:
            for d in m.moa_psi_describe_3d(*shape, dtype=dt):
                out.append((f"3d {shape} rot{rot} {dt} R={d['R']}", d, dt, int(np.prod(shape))))
    monkeypatch.setenv("MOA_FFT_PEER", "0")
    for p in (2, 8):
        sch = m.moa_dist_describe(1, p, 1 << 16, "c128")
        for d in sch["passes"]:
            out.append((f"dist1d p={p} R={d['R']}", d, "c128", (1 << 16) // p))
        sch = m.moa_dist_describe(0, p, (16, 32, 64), "c64")
        for d in sch["passes"]:
            out.append((f"dist3d p={p} R={d['R']}", d, "c64", 16 * 32 * 64 // p))
    return out


def test_kernel_movement_is_bit_exact(m, torch_cuda, monkeypatch):
    torch = torch_cuda
    checked = 0
    for name, d, dt, size in descriptors(m, monkeypatch):
        load, store, _ = enumerate_pass(d)
        span = int(max(load.max(), store.max())) + 1
        total = max(span, size)
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        x = torch.arange(total, dtype=torch.float64).to(tdt).cuda()
        y = torch.full((total,), complex(-1.0, -1.0), dtype=tdt, device="cuda")
        m.moa_pass_move(d, dt, x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        want = np.full(total, -1.0 - 1.0j)
        want[store.ravel()] = load.ravel()
        assert np.array_equal(got.astype(np.complex128), want), name
        checked += 1
    assert checked >= 30

"""GPU parity of the ablation kernels: the asynchronously fed
TMA pass kernel (MOA_FFT_WS=1: cp.async.bulk / cp.async.bulk.tensor into a ring
of shared-memory stages, mbarrier completion) and the thread-pair radix-32
kernel with the warp-shuffle exchange (MOA_FFT_PAIR=1), each against the
oracle on the same seeded inputs (BASELINE.json tolerances), and the TMA
kernel bit for bit against the plain one (same arithmetic)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-11, "c64": 2e-5}

# liftings whose passes take the variant: 512- / 1024-point lines, line-fast
# (tensor-map boxes) and contiguous (bulk copies) loads, twiddled and last passes,
# ragged multi-digit line sets
CASES_1D = [
    (1 << 20, 4, "c128", [512, 512, 4]),
    (1 << 20, 2, "c128", [1024, 1024]),
    (1 << 22, 1, "c128", [512, 1024, 8]),
    (1 << 18, 3, "c128", [512, 512]),
    (1 << 19, 1, "c128", [512, 1024]),
    (1 << 20, 3, "c64", [1024, 1024]),
    (1 << 19, 2, "c64", [512, 1024]),
]


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


def run(torch, plan, x, inverse=False):
    xt = torch.from_numpy(x).cuda()
    y = plan.exec(xt)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("env", ["MOA_FFT_WS", "MOA_FFT_PAIR"])
@pytest.mark.parametrize("n,batch,dtype,radices", CASES_1D)
def test_variant_1d_vs_oracle(m, torch_cuda, monkeypatch, env, n, batch, dtype, radices):
    monkeypatch.setenv(env, "1")
    x = synth.fill(n * batch, 31, synth.NORMAL, dtype)
    y = run(torch_cuda, m.FFTPlan(n, batch, dtype, radices=radices), x)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]


@pytest.mark.parametrize("env", ["MOA_FFT_WS", "MOA_FFT_PAIR"])
@pytest.mark.parametrize("shape,dtype,rot", [((64, 1024, 32), "c128", ""), ((32, 512, 512), "c128", "0"),
                                             ((16, 1024, 1024), "c128", ""), ((512, 8, 64), "c128", "2")])
def test_variant_3d_vs_oracle(m, torch_cuda, monkeypatch, env, shape, dtype, rot):
    monkeypatch.setenv(env, "1")
    monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
    N = int(np.prod(shape))
    x = synth.fill(N, 32, synth.NORMAL, dtype)
    y = run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype=dtype), x).reshape(shape)
    ref = oracle.fft3d(x.astype(np.complex128).reshape(shape))
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]


@pytest.mark.parametrize("env", ["MOA_FFT_WS", "MOA_FFT_PAIR"])
def test_variant_inverse_normalized(m, torch_cuda, monkeypatch, env):
    monkeypatch.setenv(env, "1")
    n, b = 1 << 19, 2
    x = synth.fill(n * b, 33, synth.UNIFORM, "c128")
    y = run(torch_cuda, m.FFTPlan(n, b, "c128", inverse=True, normalize=True), x)
    ref = oracle.fft_radix2_rows_sign(x, n, +1) / n
    assert rel_l2(y, ref) <= 1e-11


def test_ws_bitexact_vs_plain(m, torch_cuda, monkeypatch):
    # the TMA-fed kernel runs the plain kernel's arithmetic on the landed tile
    x = synth.fill((1 << 20) * 4, 34, synth.NORMAL, "c128")
    outs = []
    for ws in ("0", "1"):
        monkeypatch.setenv("MOA_FFT_WS", ws)
        outs.append(run(torch_cuda, m.FFTPlan(1 << 20, 4, "c128", radices=[512, 512, 4]), x))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.slow
@pytest.mark.parametrize("env", ["MOA_FFT_WS", "MOA_FFT_PAIR"])
def test_variant_cfg3_full(m, torch_cuda, monkeypatch, env):
    # BASELINE.json cfg3 (2^28 complex128, the planner's 512*512*1024 lifting),
    # whole-vector rel-L2 against the oracle
    monkeypatch.setenv(env, "1")
    n = synth.CONFIGS["cfg3"]["n"]
    x = synth.config_input("cfg3")
    y = run(torch_cuda, m.FFTPlan(n, 1, "c128"), x)
    ref = oracle.fft_radix2(x)
    assert rel_l2(y, ref) <= 1e-11


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("t,batch", [(6, 1), (7, 3), (8, 1), (9, 64), (10, 1), (10, 7), (11, 2), (12, 5)])
def test_small_kernel_vs_oracle_and_plain(m, torch_cuda, monkeypatch, dtype, t, batch):
    # the latency form of one-pass plans with few lines (cfg1's 2^10), forward
    # and inverse-normalised, against the oracle and the throughput kernel
    n = 1 << t
    x = synth.fill(n * batch, 35, synth.UNIFORM, dtype)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    monkeypatch.setenv("MOA_FFT_SMALL", "1")
    y = run(torch_cuda, m.FFTPlan(n, batch, dtype), x)
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]
    yi = run(torch_cuda, m.FFTPlan(n, batch, dtype, inverse=True, normalize=True), x)
    refi = oracle.fft_radix2_rows_sign(x.astype(np.complex128), n, +1) / n
    assert rel_l2(yi.astype(np.complex128), refi) <= TOL[dtype]
    monkeypatch.setenv("MOA_FFT_SMALL", "0")
    y0 = run(torch_cuda, m.FFTPlan(n, batch, dtype), x)
    assert rel_l2(y.astype(np.complex128), y0.astype(np.complex128)) <= TOL[dtype]


# TMA store of the transposed side (MOA_FFT_TMA_ST=1, pass_kernel_st): the
# complex128 512- / 1024-point passes with contiguous loads and line-fast
# stores (1-D last passes, every 3-D rotating pass) stage the tile in shared
# memory and write it with tensor-map boxes.  Same arithmetic, so bit for bit
# against the plain stores; and against the oracle.
TMA_ST_1D = [(1 << 20, 1, None), (1 << 19, 4, None), (1 << 18, 2, None), (1 << 20, 2, [1024, 1024]),
             (1 << 22, 1, [512, 1024, 8])]
TMA_ST_3D = [(64, 64, 1024), (16, 512, 1024), (8, 1024, 512)]


@pytest.mark.parametrize("n,batch,radices", TMA_ST_1D)
def test_tma_store_1d(m, torch_cuda, monkeypatch, n, batch, radices):
    x = synth.fill(n * batch, 41, synth.NORMAL, "c128")
    mk = (lambda: m.FFTPlan(n, batch, "c128", radices=radices)) if radices else (lambda: m.FFTPlan(n, batch, "c128"))
    monkeypatch.setenv("MOA_FFT_TMA_ST", "0")
    y0 = run(torch_cuda, mk(), x)
    monkeypatch.setenv("MOA_FFT_TMA_ST", "1")
    y1 = run(torch_cuda, mk(), x)
    assert np.array_equal(y0, y1)
    ref = oracle.fft_radix2_rows(x, n)
    assert rel_l2(y1, ref) <= TOL["c128"]
    yi = run(torch_cuda, m.FFTPlan(n, batch, "c128", inverse=True, normalize=True), x)
    refi = oracle.fft_radix2_rows_sign(x, n, +1) / n
    assert rel_l2(yi, refi) <= TOL["c128"]


@pytest.mark.parametrize("shape", TMA_ST_3D)
def test_tma_store_3d(m, torch_cuda, monkeypatch, shape):
    N = shape[0] * shape[1] * shape[2]
    x = synth.fill(N, 43, synth.NORMAL, "c128")
    monkeypatch.setenv("MOA_FFT_TMA_ST", "0")
    y0 = run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype="c128"), x)
    monkeypatch.setenv("MOA_FFT_TMA_ST", "1")
    y1 = run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype="c128"), x)
    assert np.array_equal(y0, y1)
    ref = oracle.fft3d(x.reshape(shape)).reshape(-1)
    assert rel_l2(y1, ref) <= TOL["c128"]


@pytest.mark.parametrize("wname", ["cfg3", "cfg5"])
def test_tma_store_full_size_bit_exact(m, torch_cuda, monkeypatch, wname):
    # BASELINE.json cfg3 (2^28) / cfg5 (1024^3) at full size, on the device:
    # the TMA-store plan bit for bit against the plain-store plan (the plain
    # plan's whole-vector parity against the oracle is tests/test_gpu_parity.py)
    torch = torch_cuda
    c = synth.CONFIGS[wname]
    x = torch.from_numpy(synth.config_input(wname)).cuda()
    mk = (lambda: m.FFTPlan.plan_3d(*c["shape"], dtype="c128")) if wname == "cfg5" else \
        (lambda: m.FFTPlan(c["n"], 1, "c128"))
    monkeypatch.setenv("MOA_FFT_TMA_ST", "0")
    y0 = mk().exec(x)
    monkeypatch.setenv("MOA_FFT_TMA_ST", "1")
    y1 = mk().exec(x)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(y0), torch.view_as_real(y1))


@pytest.mark.parametrize("n,batch,radices", [(1 << 20, 1, None), (1 << 19, 4, [512, 1024]), (1 << 20, 2, [1024, 1024])])
def test_tma_store_c64(m, torch_cuda, monkeypatch, n, batch, radices):
    # the complex64 form (MOA_FFT_TMA_ST=1): bit for bit against plain stores
    x = synth.fill(n * batch, 47, synth.NORMAL, "c64")
    mk = (lambda: m.FFTPlan(n, batch, "c64", radices=radices)) if radices else (lambda: m.FFTPlan(n, batch, "c64"))
    monkeypatch.setenv("MOA_FFT_TMA_ST", "0")
    y0 = run(torch_cuda, mk(), x)
    monkeypatch.setenv("MOA_FFT_TMA_ST", "1")
    y1 = run(torch_cuda, mk(), x)
    assert np.array_equal(y0, y1)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    assert rel_l2(y1.astype(np.complex128), ref) <= TOL["c64"]


@pytest.mark.parametrize("shape", [(64, 64, 1024), (16, 512, 1024)])
def test_tma_store_3d_c64(m, torch_cuda, monkeypatch, shape):
    N = shape[0] * shape[1] * shape[2]
    x = synth.fill(N, 49, synth.NORMAL, "c64")
    monkeypatch.setenv("MOA_FFT_TMA_ST", "0")
    y0 = run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype="c64"), x)
    monkeypatch.setenv("MOA_FFT_TMA_ST", "1")
    y1 = run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype="c64"), x)
    assert np.array_equal(y0, y1)
    ref = oracle.fft3d(x.astype(np.complex128).reshape(shape)).reshape(-1)
    assert rel_l2(y1.astype(np.complex128), ref) <= TOL["c64"]

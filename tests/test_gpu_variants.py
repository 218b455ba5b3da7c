"""GPU parity of the plan variants (include/moa_fft.h plan flags; SURVEY.md
§8(f) f1, f3): the inverse sign e^{+2 pi i jk/n} (the fftpsirad2 fragment's
EXP(+2 pi i row/L)), the 1/N normalisation, and the lifted output order
(the final transpose left undone) with its exported index map.
Reference: the oracle (oracle/) on the same seeded inputs."""
import numpy as np
import pytest

import oracle
import synth
from oracle import moa

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-11, "c64": 2e-5}


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


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(torch, plan, x):
    xt = torch.from_numpy(x).cuda()
    y = plan.exec(xt)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,batch", [(1, 3), (16, 2), (1 << 10, 1), (1 << 13, 3), (1 << 16, 2), (1 << 20, 1)])
@pytest.mark.parametrize("normalize", [False, True])
def test_inverse_1d(m, torch_cuda, dtype, n, batch, normalize):
    x = synth.fill(n * batch, 50 + n % 97, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype, inverse=True, normalize=normalize)
    y = run(torch_cuda, plan, x).astype(np.complex128)
    ref = oracle.fft_radix2_rows_sign(x.astype(np.complex128), n, +1)
    if normalize:
        ref = ref / n
    assert rel_l2(y, ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_forward_normalized_and_roundtrip(m, torch_cuda, dtype):
    n, batch = 1 << 14, 2
    x = synth.fill(n * batch, 61, synth.NORMAL, dtype)
    fwd = m.FFTPlan(n, batch, dtype, normalize=True)
    inv = m.FFTPlan(n, batch, dtype, inverse=True)
    X = run(torch_cuda, fwd, x)
    assert rel_l2(X.astype(np.complex128), oracle.fft_radix2_rows(x.astype(np.complex128), n) / n) <= TOL[dtype]
    back = run(torch_cuda, inv, X)                       # (1/n) F then F^{-1} unnormalised = identity
    assert rel_l2(back.astype(np.complex128), x.astype(np.complex128)) <= TOL[dtype]


@pytest.mark.parametrize("shape", [(8, 16, 32), (64, 32, 16)])
def test_inverse_3d(m, torch_cuda, shape):
    x = synth.fill(int(np.prod(shape)), 71, synth.NORMAL).reshape(shape)
    plan = m.FFTPlan.plan_3d(*shape, dtype="c128", inverse=True, normalize=True)
    y = run(torch_cuda, plan, x.reshape(-1)).reshape(shape)
    ref = oracle.fft3d_sign(x, +1) / x.size
    assert rel_l2(y, ref) <= 1e-11


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,batch", [(1 << 10, 2), (1 << 13, 3), (1 << 14, 3), (1 << 16, 2), (1 << 20, 1),
                                     (1 << 24, 1)])
def test_lifted_order_1d(m, torch_cuda, dtype, n, batch):
    # (2^14 complex128 rows are a cluster pair in natural order; lifted order
    # takes the plain two-pass form)
    x = synth.fill(n * batch, 81, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype, lifted_order=True)
    pos = plan.output_index()
    assert np.array_equal(np.sort(pos), np.arange(n))          # a permutation of the row
    y = run(torch_cuda, plan, x).reshape(batch, n)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n).reshape(batch, n)
    assert rel_l2(y[:, pos].astype(np.complex128), ref) <= TOL[dtype]
    radices = [1 << d["logR"] for d in plan.describe()]
    if len(radices) > 1 and n <= (1 << 16):
        # bit-exact against the oracle's MoA materialisation: in lifted order X
        # stays at the position the last pass loaded it from, i.e. the ravel of
        # the axis-reversing transpose of <R_0 ... R_{P-1}> rho-hat iota n
        z = moa.reshape(radices, moa.iota(n))
        P = len(radices)
        T = moa.transpose(z, [P - 1 - ax for ax in range(P)])
        assert np.array_equal(pos, np.array(T.rav, dtype=np.int64))


def test_lifted_order_single_pass_is_natural(m, torch_cuda):
    plan = m.FFTPlan(1 << 10, 1, "c128", lifted_order=True)
    assert np.array_equal(plan.output_index(), np.arange(1 << 10))


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("flags", ["lifted", "inverse_norm", "lifted_inverse"])
def test_dist_1d_loopback_variants(m, torch_cuda, p, flags):
    torch = torch_cuda
    N = 1 << 18
    dtype = "c128"
    x = synth.fill(N, 5, synth.UNIFORM, dtype)
    kw = dict(lifted_order="lifted" in flags, inverse="inverse" in flags, normalize="norm" in flags)
    plans = []
    for r in range(p):
        m.moa_fft_dist_loopback(r, p)
        plans.append(m.FFTPlan(N, 1, dtype, ngpu=p, **kw))
    shards = [torch.from_numpy(s.copy()).cuda() for s in np.split(x, p)]
    outs = [torch.empty_like(s) for s in shards]
    m.moa_fft_exec_loopback([pl.h for pl in plans], [s.data_ptr() for s in shards], [o.data_ptr() for o in outs],
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    y = np.concatenate([o.cpu().numpy() for o in outs])
    ref = oracle.fft_radix2_sign(x, +1 if kw["inverse"] else -1)
    if kw["normalize"]:
        ref = ref / N
    pos = plans[0].output_index()
    assert rel_l2(y[pos], ref) <= 1e-11


def test_exec_host_inverse(m, torch_cuda):
    torch = torch_cuda
    n, batch = 1 << 12, 16                                     # batched: the chunked sub-plan pipeline
    x = synth.fill(n * batch, 91, synth.UNIFORM)
    plan = m.FFTPlan(n, batch, "c128", inverse=True, normalize=True)
    hin = torch.from_numpy(x).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    plan.exec_host(hin, hout)
    ref = oracle.fft_radix2_rows_sign(x, n, +1) / n
    assert rel_l2(hout.numpy(), ref) <= 1e-11


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,batch", [(1, 2), (2, 3), (1 << 10, 2), (1 << 17, 1)])
def test_unblocked_control(m, torch_cuda, dtype, n, batch):
    # the paper's unblocked control: P_n then t global radix-2 stages
    x = synth.fill(n * batch, 101, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype, unblocked=True)
    d = plan.describe()
    assert [p["kind"] for p in d] == [3] + [2] * (n.bit_length() - 1)
    y = run(torch_cuda, plan, x).astype(np.complex128)
    assert rel_l2(y, oracle.fft_radix2_rows(x.astype(np.complex128), n)) <= TOL[dtype]
    inv = m.FFTPlan(n, batch, dtype, unblocked=True, inverse=True, normalize=True)
    z = run(torch_cuda, inv, x).astype(np.complex128)
    assert rel_l2(z, oracle.fft_radix2_rows_sign(x.astype(np.complex128), n, +1) / n) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,batch", [(1, 3), (2, 5), (8, 3), (1 << 10, 4), (1 << 13, 1), (1 << 17, 2), (1 << 20, 1)])
def test_hypercube_form(m, torch_cuda, dtype, n, batch):
    # the Ch.5 hypercube stages with physical t_j transposes
    # (one loop over (i, i + n/2) per stage, no bit reversal), forward and
    # inverse-normalised, against the oracle
    x = synth.fill(n * batch, 36, synth.UNIFORM, dtype)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    plan = m.FFTPlan(n, batch, dtype, hypercube=True)
    d = plan.describe()
    assert n == 1 or (len(d) == int(np.log2(n)) and all(p["kind"] == 4 for p in d))
    y = run(torch_cuda, plan, x)
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]
    inv = m.FFTPlan(n, batch, dtype, hypercube=True, inverse=True, normalize=True)
    yi = run(torch_cuda, inv, x)
    refi = oracle.fft_radix2_rows_sign(x.astype(np.complex128), n, +1) / n
    assert rel_l2(yi.astype(np.complex128), refi) <= TOL[dtype]
    xt = torch_cuda.from_numpy(x).cuda()                                   # in == out: staged input
    plan.exec(xt, xt)
    torch_cuda.cuda.synchronize()
    assert rel_l2(xt.cpu().numpy().astype(np.complex128), ref) <= TOL[dtype]

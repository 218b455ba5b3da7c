"""GPU parity: the CUDA path through the C-ABI against the oracle, on the same
seeded inputs (synth/).  Tolerances are BASELINE.json's: relative L2 error
<= 1e-11 (complex128) and <= 2e-5 (complex64)."""
import numpy as np
import pytest

import oracle
import synth

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


def gpu_run(torch, plan, x: np.ndarray, inplace=False):
    xt = torch.from_numpy(x).cuda()
    out = xt if inplace else torch.empty_like(xt)
    plan.exec(xt, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def npdt(dtype):
    return np.complex128 if dtype == "c128" else np.complex64


# ---------------------------------------------------------------- cfg1
def test_cfg1_vs_direct_dft(m, torch_cuda):
    c = synth.CONFIGS["cfg1"]
    x = synth.config_input("cfg1")
    plan = m.FFTPlan(c["n"], 1, "c128")
    y = gpu_run(torch_cuda, plan, x)
    assert rel_l2(y, oracle.dft_direct(x)) <= 1e-11           # BASELINE.json: checked against O(n^2)
    assert rel_l2(y, oracle.fft_radix2(x)) <= 1e-11


# ---------------------------------------------------------------- sweeps
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("t", list(range(0, 23)))
def test_sizes_sweep(m, torch_cuda, dtype, t):
    n = 1 << t
    batch = max(1, min(5, (1 << 20) // n)) if t < 20 else 1
    x = synth.fill(n * batch, 1000 + t, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype)
    y = gpu_run(torch_cuda, plan, x)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype], (n, batch, plan.describe())


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("radices,batch", [
    ([2, 2], 3), ([2, 2, 2, 2, 2], 1), ([4, 8], 7), ([16, 16], 2), ([8, 32, 4], 1), ([512, 512], 1),
    ([4096, 2], 1), ([2, 4096], 1), ([64, 64, 64], 1), ([1024, 256], 1), ([128, 64, 16, 8], 1),
    ([2048, 2048], 1), ([32, 4096], 1), ([4096, 16], 3),
])
def test_explicit_liftings(m, torch_cuda, dtype, radices, batch):
    # the paper's run-time blocking choice, including unbalanced and
    # all-radix-2 liftings (the unblocked-control extreme)
    n = int(np.prod(radices))
    x = synth.fill(n * batch, 7, synth.NORMAL, dtype)
    plan = m.FFTPlan(n, batch, dtype, radices=radices)
    y = gpu_run(torch_cuda, plan, x)
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]


@pytest.mark.parametrize("fuse", ["1", "2", "0"])
@pytest.mark.parametrize("n,batch,dtype,radices", [
    (1 << 10, 100, "c128", [32, 32]), (1 << 16, 64, "c128", None), (1 << 12, 300, "c64", [64, 64]),
    (1 << 14, 40, "c64", [128, 128]), (1 << 11, 77, "c128", [64, 32]), (1 << 20, 17, "c64", [1024, 1024]),
])
def test_fused_pairs(m, torch_cuda, monkeypatch, fuse, n, batch, dtype, radices):
    # the L2-staged pass pair (ring slots reused many times; with and without the
    # discard of consumed lines; "0" = the unfused two-launch control)
    monkeypatch.setenv("MOA_FFT_FUSE", fuse)
    x = synth.fill(n * batch, 21, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype, radices=radices)
    d = plan.describe()
    assert (d[0]["ring"] == 2) == (fuse != "0")
    for rep in range(3):                                   # epochs advance across execs
        y = gpu_run(torch_cuda, plan, x)
        ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
        assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype], rep


@pytest.mark.parametrize("n,batch,dtype,radices", [
    (1 << 20, 3, "c128", [32, 32, 32, 32]), (1 << 22, 2, "c64", [64, 64, 32, 32]),
    (1 << 24, 1, "c128", [64, 64, 64, 64]), (1 << 24, 1, "c64", [64, 64, 64, 64]),
    (1 << 26, 1, "c64", [128, 128, 64, 64]),
])
def test_lift4_fused_pairs(m, torch_cuda, monkeypatch, n, batch, dtype, radices):
    # large single transforms: four factors as two L2-staged pairs (two HBM round trips)
    monkeypatch.setenv("MOA_FFT_LIFT4", "1")
    x = synth.fill(n * batch, 22, synth.NORMAL, dtype)
    plan = m.FFTPlan(n, batch, dtype, radices=radices)
    assert [d["ring"] for d in plan.describe()] == [2, 1, 2, 1]
    for rep in range(2):
        y = gpu_run(torch_cuda, plan, x)
        ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
        assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype], rep


# ---------------------------------------------------------------- edge cases
def test_identity_and_tiny(m, torch_cuda):
    for dtype in ("c128", "c64"):
        x = synth.fill(37, 3, synth.UNIFORM, dtype)
        y = gpu_run(torch_cuda, m.FFTPlan(1, 37, dtype), x)               # n = 1: identity (t = 0)
        assert np.array_equal(y, x)
        x = synth.fill(2 * 1001, 3, synth.UNIFORM, dtype)
        y = gpu_run(torch_cuda, m.FFTPlan(2, 1001, dtype), x)
        ref = np.stack([x[0::2] + x[1::2], x[0::2] - x[1::2]], axis=1).reshape(-1)
        assert rel_l2(y, ref) <= TOL[dtype]


def test_in_place_and_determinism(m, torch_cuda, monkeypatch):
    plans = [(lambda n=n, b=b: m.FFTPlan(n, b, "c128"), n * b) for n, b in [(1 << 10, 4), (1 << 16, 3), (1 << 21, 1)]]
    plans += [(lambda: m.FFTPlan(1 << 12, 2, "c128", unblocked=True), 1 << 13),      # gather (bit reversal) first
              (lambda: m.FFTPlan(1 << 14, 2, "c128", lifted_order=True), 1 << 15),
              (lambda: m.FFTPlan.plan_3d(16, 32, 64, "c128"), 16 * 32 * 64),          # rotating layouts
              (lambda: m.FFTPlan.plan_3d(16, 32, 64, "c64"), 16 * 32 * 64)]
    for make, size in plans:
        plan = make()
        dt = "c64" if plan.dtype == m.MOA_C64 else "c128"
        x = synth.fill(size, 11, synth.UNIFORM, dt)
        y1 = gpu_run(torch_cuda, plan, x)
        y2 = gpu_run(torch_cuda, plan, x, inplace=True)
        y3 = gpu_run(torch_cuda, plan, x)
        assert np.array_equal(y1, y2) and np.array_equal(y1, y3)      # bitwise deterministic, in-place ok


def test_exec_rejects_bad_pointers(m, torch_cuda):
    torch = torch_cuda
    plan = m.FFTPlan(1024, 1, "c128")
    buf = torch.empty(2048 + 1, dtype=torch.complex64, device="cuda")
    with pytest.raises(m.MoaError) as ei:
        m.moa_fft_exec(plan.h, buf.data_ptr() + 8, buf.data_ptr() + 8, 0)    # 8-byte aligned only
    assert ei.value.status == m.MOA_EINVAL
    with pytest.raises(m.MoaError):
        m.moa_fft_exec(plan.h, 0, buf.data_ptr(), 0)


def test_closed_forms_large(m, torch_cuda):
    n = 1 << 22
    d = np.zeros(n, np.complex128)
    d[0] = 1
    y = gpu_run(torch_cuda, m.FFTPlan(n, 1, "c128"), d)
    assert np.max(np.abs(y - 1)) < 1e-12
    k0 = 123457
    j = np.arange(n)
    e = np.exp(2j * np.pi * ((k0 * j) % n) / n)
    y = gpu_run(torch_cuda, m.FFTPlan(n, 1, "c128"), e)
    assert abs(y[k0] - n) < 1e-6
    y[k0] = 0
    assert np.max(np.abs(y)) < 1e-6


def test_exec_host_e2e(m, torch_cuda):
    torch = torch_cuda
    n, batch = 1 << 14, 8
    x = synth.fill(n * batch, 12, synth.UNIFORM)
    plan = m.FFTPlan(n, batch, "c128")
    hin = torch.from_numpy(x).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    plan.exec_host(hin, hout)
    assert rel_l2(hout.numpy(), oracle.fft_radix2_rows(x, n)) <= 1e-11


# ---------------------------------------------------------------- 3-D
@pytest.mark.parametrize("shape,dtype,rot", [((8, 1024, 1024), "c64", ""), ((8, 1024, 512), "c64", "0"),
                                             ((16, 512, 256), "c64", "0")])
def test_3d_fused_wide_planes(m, torch_cuda, monkeypatch, shape, dtype, rot):
    # fused z/y pair whose y-pass tiles are narrower than a 128-byte line
    # (W * esize < 128): the L2 discard of consumed ring lines must not drop
    # lines of the neighbouring tile; several executions, so the
    # per-launch counter reset is exercised too
    monkeypatch.setenv("MOA_FFT_FUSE", "1")
    monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
    N = int(np.prod(shape))
    x = synth.fill(N, 14, synth.NORMAL, dtype)
    plan = m.FFTPlan.plan_3d(*shape, dtype=dtype)
    ref = oracle.fft3d(x.astype(np.complex128).reshape(shape))
    for rep in range(3):
        y = gpu_run(torch_cuda, plan, x).reshape(shape)
        assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype], rep


@pytest.mark.parametrize("shape", [(8, 8, 8), (4, 16, 32), (64, 32, 16), (2, 2, 2), (1, 8, 4), (128, 128, 128)])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("fuse,rot", [("", ""), ("1", "0"), ("", "0"), ("", "1"), ("", "2"), ("", "3")])
def test_3d(m, torch_cuda, monkeypatch, shape, dtype, fuse, rot):
    monkeypatch.setenv("MOA_FFT_FUSE", fuse)
    monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
    N = int(np.prod(shape))
    x = synth.fill(N, 13, synth.NORMAL, dtype)
    plan = m.FFTPlan.plan_3d(*shape, dtype=dtype)
    y = gpu_run(torch_cuda, plan, x).reshape(shape)
    ref = oracle.fft3d(x.astype(np.complex128).reshape(shape))
    assert rel_l2(y.astype(np.complex128), ref) <= TOL[dtype]


# ---------------------------------------------------------------- loopback processor lifting
@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_dist_1d_loopback(m, torch_cuda, monkeypatch, p, dtype, peer):
    # peer 1: E2 and E3 fused into the stores of pass A / the last local pass
    # (every virtual rank's kernel writes straight into the others' buffers)
    monkeypatch.setenv("MOA_FFT_PEER", peer)
    torch = torch_cuda
    N = 1 << 20
    x = synth.fill(N, 3, synth.UNIFORM, dtype)
    plans = []
    for r in range(p):
        m.moa_fft_dist_loopback(r, p)
        plans.append(m.FFTPlan(N, 1, dtype, ngpu=p))
    shards = [torch.from_numpy(s.copy()).cuda() for s in np.split(x, p)]
    outs = [torch.empty_like(s) for s in shards]
    m.moa_fft_exec_loopback([pl.h for pl in plans], [s.data_ptr() for s in shards], [o.data_ptr() for o in outs],
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    y = np.concatenate([o.cpu().numpy() for o in outs]).astype(np.complex128)
    ref = oracle.fft_radix2(x.astype(np.complex128))
    assert rel_l2(y, ref) <= TOL[dtype]


@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_3d_loopback(m, torch_cuda, monkeypatch, p, peer):
    monkeypatch.setenv("MOA_FFT_PEER", peer)
    torch = torch_cuda
    shape = (64, 32, 16)
    x = synth.fill(int(np.prod(shape)), 4, synth.NORMAL).reshape(shape)
    plans = []
    for r in range(p):
        m.moa_fft_dist_loopback(r, p)
        plans.append(m.FFTPlan.plan_3d(*shape, dtype="c128", ngpu=p))
    shards = [torch.from_numpy(np.ascontiguousarray(s).reshape(-1)).cuda() for s in np.split(x, p, axis=0)]
    outs = [torch.empty_like(s) for s in shards]
    m.moa_fft_exec_loopback([pl.h for pl in plans], [s.data_ptr() for s in shards], [o.data_ptr() for o in outs],
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = oracle.fft3d(x)
    n1l = shape[1] // p
    for r in range(p):
        want = ref[:, r * n1l:(r + 1) * n1l, :].reshape(-1)
        assert rel_l2(outs[r].cpu().numpy(), want) <= 1e-11


# ---------------------------------------------------------------- BASELINE.json full sizes
def _sample_bins(n, count, seed):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, n // 2, n - 1, n // 3]
    return np.unique(np.concatenate([fixed, rng.integers(0, n, count)]).astype(np.int64))


def test_cfg2_full(m, torch_cuda):
    c = synth.CONFIGS["cfg2"]
    n, b = c["n"], c["batch"]
    x = synth.config_input("cfg2")
    y = gpu_run(torch_cuda, m.FFTPlan(n, b, "c128"), x)
    ref = oracle.fft_radix2_rows(x, n)                      # the whole 1 GiB against the oracle
    assert rel_l2(y, ref) <= 1e-11


def rel_l2_chunked(y, ref, chunk=1 << 26):
    """rel-L2 in double over chunks (no full-size temporaries)."""
    num = den = 0.0
    for s in range(0, ref.size, chunk):
        r = ref[s:s + chunk]
        d = y[s:s + chunk].astype(np.complex128) - r
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(r, r).real)
    return float(np.sqrt(num / den))


def _sampled_bins_check(x, y, n, bins, tol):
    ref = oracle.dft_bins(x, n, bins)
    scale = np.sqrt(n) * np.sqrt(np.mean(np.abs(x.astype(np.complex128)) ** 2))   # |X[k]| ~ sqrt(n) rms(x)
    assert np.max(np.abs(y[bins].astype(np.complex128) - ref)) / scale <= tol


# Whole-vector parity at BASELINE.json's full sizes: the GPU output against the
# oracle's radix-2 FFT (O1+O2; O5 for 3-D) of the same seeded input, every
# element, rel-L2 at BASELINE.json's tolerance (Van Loan "Output: The FFT of x",
# P:1849-1852).  The sampled bins against the O(n^2) definition stay as an
# independent second pin.
@pytest.mark.slow
def test_cfg3_full(m, torch_cuda):
    n = synth.CONFIGS["cfg3"]["n"]
    x = synth.config_input("cfg3")
    y = gpu_run(torch_cuda, m.FFTPlan(n, 1, "c128"), x)
    _sampled_bins_check(x, y, n, _sample_bins(n, 6, 2), 1e-11)
    ref = oracle.fft_radix2(x)
    del x
    err = rel_l2_chunked(y, ref)
    print(f"cfg3 whole-vector rel-L2 {err:.3e}")
    assert err <= 1e-11


@pytest.mark.slow
def test_cfg4_full(m, torch_cuda):
    n = synth.CONFIGS["cfg4"]["n"]
    x = synth.config_input("cfg4")
    y = gpu_run(torch_cuda, m.FFTPlan(n, 1, "c64"), x)
    _sampled_bins_check(x, y, n, _sample_bins(n, 4, 3), 2e-5)
    ref = x.astype(np.complex128)                 # complex64 promoted exactly
    del x
    oracle.fft_radix2_inplace(ref)
    err = rel_l2_chunked(y, ref)
    print(f"cfg4 whole-vector rel-L2 {err:.3e}")
    assert err <= 2e-5


@pytest.mark.slow
def test_cfg5_full(m, torch_cuda):
    shape = synth.CONFIGS["cfg5"]["shape"]
    x = synth.config_input("cfg5")
    y = gpu_run(torch_cuda, m.FFTPlan.plan_3d(*shape, dtype="c128"), x)
    rng = np.random.default_rng(4)
    ks = np.array([(0, 0, 0), (1, 2, 3), (1023, 512, 7)] + [tuple(rng.integers(0, 1024, 3)) for _ in range(2)],
                  dtype=np.int64)
    ref_b = oracle.dft3_bins(x, shape, ks)
    got = y.reshape(shape)[ks[:, 0], ks[:, 1], ks[:, 2]]
    N = int(np.prod(shape))
    scale = np.sqrt(N) * np.sqrt(np.mean(np.abs(x) ** 2))
    assert np.max(np.abs(got - ref_b)) / scale <= 1e-11
    ref = x.reshape(shape)
    del x
    oracle.fft3d_inplace(ref)
    err = rel_l2_chunked(y, ref.reshape(-1))
    print(f"cfg5 whole-vector rel-L2 {err:.3e}")
    assert err <= 1e-11


@pytest.mark.parametrize("radices,wpass", [([256, 512, 2048], "2:4"), ([1024, 1024, 256], "0:8,1:8")])
def test_c64_wide_tiles_bit_exact(m, torch_cuda, monkeypatch, radices, wpass):
    """Round 2 session 2's complex64 tile rules (16-line tiles for 1024-point
    line-coalesced passes; 8-line 1024-thread tiles for >= 2^11-point passes
    storing >= 1 MiB apart) change only which lines share a CTA, so the result
    is bit-identical to the narrower tiles (MOA_FFT_W_PASS), and on sampled
    bins within the tolerance of the oracle's definition."""
    n = 1 << 28
    x = synth.fill(n, 23, synth.UNIFORM, "c64")
    wide = m.FFTPlan(n, 1, "c64", radices=radices)
    monkeypatch.setenv("MOA_FFT_W_PASS", wpass)
    narrow = m.FFTPlan(n, 1, "c64", radices=radices)
    ww, wn = [d["W"] for d in wide.describe()], [d["W"] for d in narrow.describe()]
    assert ww != wn and max(d["threads"] for d in wide.describe()) >= 512
    y = gpu_run(torch_cuda, wide, x)
    y2 = gpu_run(torch_cuda, narrow, x)
    assert np.array_equal(y.view(np.uint8), y2.view(np.uint8))
    bins = np.array([0, 1, 2047, 1 << 17, (1 << 20) + 3, n // 2, n - 1], dtype=np.int64)
    _sampled_bins_check(x, y, n, bins, 2e-5)

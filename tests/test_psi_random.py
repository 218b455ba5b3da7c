"""Property-based tests of the psi-index layer (CPU): for random liftings
n = R_0 ... R_{P-1}, batches, dtypes and 3-D shapes, the ONF descriptors the
library emits -- executed by the test-side numpy interpreter of the ONF
semantics in include/moa_fft.h -- reproduce the oracle's DFT, and every pass
is a permutation of the array (each element loaded once and stored once)."""
import numpy as np
from hypothesis import given, settings, strategies as st

import oracle
import synth
from onf import enumerate_pass, run_plan

import paper_0803_2386_b200 as m


@st.composite
def liftings(draw):
    t = draw(st.integers(min_value=1, max_value=13))
    nparts = draw(st.integers(min_value=1, max_value=min(t, 6)))
    cuts = sorted(draw(st.lists(st.integers(min_value=1, max_value=t - 1), min_size=nparts - 1,
                                max_size=nparts - 1, unique=True))) if nparts > 1 and t > 1 else []
    bits, prev = [], 0
    for c in cuts + [t]:
        bits.append(c - prev)
        prev = c
    out = []
    for b in bits:                      # each radix <= 2^12 (one CTA line)
        while b > 12:
            out.append(12)
            b -= 12
        if b > 0:
            out.append(b)
    return [1 << b for b in out]


@settings(max_examples=60, deadline=None)
@given(radices=liftings(), batch=st.integers(min_value=1, max_value=3), dtype=st.sampled_from(["c128", "c64"]))
def test_random_liftings_compute_the_dft(radices, batch, dtype):
    n = int(np.prod(radices))
    passes = m.moa_psi_describe(n, batch, dtype, radices)
    x = synth.fill(n * batch, 31, synth.UNIFORM)
    got = run_plan(passes, x)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    for d in passes:
        load, store, _ = enumerate_pass(d)
        if not d.get("ring", 0):
            assert np.array_equal(np.sort(load.ravel()), np.arange(n * batch))
            assert np.array_equal(np.sort(store.ravel()), np.arange(n * batch))
        assert d["threads"] <= 512 and d["W"] >= 1 and (d["ext"][0] % d["W"] == 0 if d["ndig"] else True)


@settings(max_examples=30, deadline=None)
@given(l0=st.integers(0, 6), l1=st.integers(0, 6), l2=st.integers(0, 6), dtype=st.sampled_from(["c128", "c64"]))
def test_random_3d_shapes_compute_the_dft(l0, l1, l2, dtype):
    shape = (1 << l0, 1 << l1, 1 << l2)
    passes = m.moa_psi_describe_3d(*shape, dtype=dtype)
    x = synth.fill(int(np.prod(shape)), 32, synth.NORMAL)
    got = run_plan(passes, x).reshape(shape)
    ref = oracle.fft3d(x.reshape(shape))
    assert np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300) < 1e-12


# ---------------------------------------------------------------- the kernels on random liftings (GPU)
import pytest  # noqa: E402


@pytest.mark.gpu
@settings(max_examples=40, deadline=None)
@given(radices=liftings(), batch=st.integers(min_value=1, max_value=4), dtype=st.sampled_from(["c128", "c64"]))
def test_random_liftings_on_gpu(radices, batch, dtype):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = int(np.prod(radices))
    x = synth.fill(n * batch, 33, synth.UNIFORM, dtype)
    plan = m.FFTPlan(n, batch, dtype, radices=radices)
    y = plan.exec(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    got = y.cpu().numpy().astype(np.complex128)
    tol = 1e-11 if dtype == "c128" else 2e-5
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol


# ---------------------------------------------------------------- processor-level lifting, random
@settings(max_examples=25, deadline=None)
@given(p=st.sampled_from([2, 4, 8]), t=st.integers(min_value=6, max_value=14),
       lifted=st.booleans(), peer=st.sampled_from(["0", "1"]), dtype=st.sampled_from(["c128", "c64"]))
def test_random_distributed_schedules(p, t, lifted, peer, dtype):
    import os
    from onf import run_dist
    N = 1 << t
    if N < p * p:
        return
    old = os.environ.get("MOA_FFT_PEER")
    os.environ["MOA_FFT_PEER"] = peer
    try:
        flags = m.MOA_FFT_LIFTED_ORDER if lifted else 0
        sch = [m.moa_dist_describe(r, p, N, dtype, flags=flags) for r in range(p)]
    finally:
        if old is None:
            os.environ.pop("MOA_FFT_PEER", None)
        else:
            os.environ["MOA_FFT_PEER"] = old
    x = synth.fill(N, 34, synth.UNIFORM)
    outs = run_dist(sch, np.split(x, p))
    ref = oracle.fft_radix2(x)
    for g in range(p):
        want = ref[g::p] if lifted else ref[g * (N // p):(g + 1) * (N // p)]
        assert np.linalg.norm(outs[g] - want) / np.linalg.norm(want) < 1e-12

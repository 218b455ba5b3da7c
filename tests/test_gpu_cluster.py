"""GPU parity of the cluster level of the lifting (kernels.cu cluster_kernel,
psi.cpp psi_cluster_pair): a two-pass lifting of independent rows whose row
fits one thread-block cluster's shared memory runs as one launch, pass A's
result going straight into the shared memory of the CTA that runs pass B's
tile (the reshape-transpose of Eq. reshape3, between SMs; the
block-per-hierarchy-level premise).

The arithmetic is the plain passes' (the same tile code), so the cluster plan
must be bit-identical to the two-pass plan on the same input, and within the
BASELINE tolerance of the oracle (oracle/)."""
import os

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


def plan_with(m, mode, *args, **kw):
    old = os.environ.get("MOA_FFT_CLUSTER")
    os.environ["MOA_FFT_CLUSTER"] = mode
    try:
        return m.FFTPlan(*args, **kw)
    finally:
        if old is None:
            del os.environ["MOA_FFT_CLUSTER"]
        else:
            os.environ["MOA_FFT_CLUSTER"] = old


def rings(plan):
    return [d["ring"] for d in plan.describe()]


CASES = [  # (n, batch, dtype): two-pass liftings, cluster sizes 2 .. 16
    (1 << 16, 4, "c128"),
    (1 << 16, 37, "c128"),
    (1 << 14, 9, "c128"),
    (1 << 13, 5, "c128"),
    (1 << 16, 6, "c64"),
    (1 << 14, 3, "c64"),
    (1 << 17, 2, "c64"),
]


@pytest.mark.parametrize("n,batch,dtype", CASES)
def test_cluster_pair_bit_exact_and_oracle(m, torch_cuda, n, batch, dtype):
    torch = torch_cuda
    x = synth.fill(n * batch, 70 + batch, synth.UNIFORM, dtype)
    pc = plan_with(m, "1", n, batch, dtype)
    pp = plan_with(m, "0", n, batch, dtype)
    if rings(pc) != [3, 4]:
        pytest.skip(f"no cluster pair for this lifting: {rings(pc)}")
    assert pc.launches == 1 and pp.launches == 2
    xt = torch.from_numpy(x).cuda()
    yc = pc.exec(xt).cpu().numpy()
    yp = pp.exec(xt).cpu().numpy()
    assert np.array_equal(yc.view(np.uint8), yp.view(np.uint8)), "cluster pair differs from the two passes"
    ref = oracle.fft_radix2_rows(x.astype(np.complex128), n)
    assert rel_l2(yc.astype(np.complex128), ref) <= TOL[dtype]


def test_cluster_pair_cfg2_shape(m, torch_cuda):
    """The cfg2 lifting (256 x 256, 16-CTA clusters) on 64 rows, plus an in-place exec."""
    torch = torch_cuda
    n, batch = 1 << 16, 64
    x = synth.fill(n * batch, 1, synth.UNIFORM)
    pc = plan_with(m, "1", n, batch, "c128")
    d = pc.describe()
    assert [e["ring"] for e in d] == [3, 4] and d[0]["ring_slots"] == 16 and d[0]["ring_G"] == n
    xt = torch.from_numpy(x).cuda()
    y = pc.exec(xt).cpu().numpy()
    ref = oracle.fft_radix2_rows(x, n)
    assert rel_l2(y, ref) <= 1e-11
    pc.exec(xt, xt)  # in place: each cluster reads its whole row before any store
    assert np.array_equal(xt.cpu().numpy().view(np.uint8), y.view(np.uint8))


def test_cluster_pair_default_for_small_clusters(m, torch_cuda):
    """By default the cluster level is used where a row spreads over <= 8 CTAs
    (2^14-point complex128 rows), not for cfg2's 16-CTA rows."""
    old = os.environ.pop("MOA_FFT_CLUSTER", None)
    try:
        p14 = m.FFTPlan(1 << 14, 5, "c128")
        p16 = m.FFTPlan(1 << 16, 5, "c128")
        assert rings(p14) == [3, 4] and p14.describe()[0]["ring_slots"] == 8 and p14.launches == 1
        assert rings(p16) == [0, 0] and p16.launches == 2
        x = synth.fill((1 << 14) * 5, 79, synth.UNIFORM)
        y = p14.exec(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, oracle.fft_radix2_rows(x, 1 << 14)) <= 1e-11
    finally:
        if old is not None:
            os.environ["MOA_FFT_CLUSTER"] = old


@pytest.mark.parametrize("normalize", [False, True])
def test_cluster_pair_inverse(m, torch_cuda, normalize):
    torch = torch_cuda
    n, batch = 1 << 16, 3
    x = synth.fill(n * batch, 77, synth.NORMAL)
    old = os.environ.get("MOA_FFT_CLUSTER")
    os.environ["MOA_FFT_CLUSTER"] = "1"
    try:
        plan = m.FFTPlan(n, batch, "c128", inverse=True, normalize=normalize)
    finally:
        if old is None:
            del os.environ["MOA_FFT_CLUSTER"]
        else:
            os.environ["MOA_FFT_CLUSTER"] = old
    assert rings(plan) == [3, 4]
    y = plan.exec(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = oracle.fft_radix2_rows_sign(x, n, +1)
    if normalize:
        ref = ref / n
    assert rel_l2(y, ref) <= 1e-11

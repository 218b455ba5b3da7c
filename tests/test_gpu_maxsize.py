"""The largest single transforms that fit one B200 with in, out and scratch
resident (complex64 n = 2^32, complex128 n = 2^31: 32 GiB per buffer) -- where
64-bit offsets and grid sizes matter -- checked against the closed form of a
shifted impulse: x = delta_{j0} -> X[k] = e^{-2 pi i j0 k / n} (exponent reduced
in integers), on sampled bins, plus the unit-modulus property on a slice."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("t,dtype,tol", [(32, "c64", 2e-5), (31, "c128", 1e-11)])
def test_impulse_at_maximum_size(t, dtype, tol):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0803_2386_b200 as m
    n = 1 << t
    free, _ = torch.cuda.mem_get_info()
    esize = 8 if dtype == "c64" else 16
    if free < 3.3 * n * esize:
        pytest.skip("not enough device memory for in + out + scratch")
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    j0 = n // 2 + 123457                                    # an offset beyond 2^31 elements
    plan = m.FFTPlan(n, 1, dtype)
    x = torch.zeros(n, dtype=tdt, device="cuda")
    x[j0] = 1
    y = plan.exec(x)
    del x
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    ks = np.unique(np.concatenate([[0, 1, 2, n // 2, n - 1, n - 2, (1 << 31) + 7],
                                   rng.integers(0, n, 200)]) % n).astype(np.int64)
    got = y[torch.from_numpy(ks).cuda()].cpu().numpy().astype(np.complex128)
    e = (ks.astype(object) * j0) % n                        # exact integer exponent
    want = np.exp(-2j * np.pi * np.array([float(v) for v in e]) / n)
    assert np.max(np.abs(got - want)) <= tol * np.sqrt(t)
    mod = y[: 1 << 20].abs().double().cpu().numpy()
    assert np.max(np.abs(mod - 1.0)) <= tol * np.sqrt(t)
    plan.close()

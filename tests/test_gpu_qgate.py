"""GPU parity of the Ch.6 density-matrix gate against the
oracle (oracle/qgate.py): the dense definition U_full D U_full^dagger for
small n, and -- at sizes where the dense product is out of reach -- sampled
view blocks recomputed from the original matrix through the oracle's Eq.
generic addressing."""
import numpy as np
import pytest

from oracle import qgate

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


def rand_case(n, q, seed):
    rng = np.random.default_rng(seed)
    bits = [int(b) for b in rng.choice(n, q, replace=False)]
    U, _ = np.linalg.qr(rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q)))
    M = rng.standard_normal((1 << n, 1 << n)) + 1j * rng.standard_normal((1 << n, 1 << n))
    D = M @ M.conj().T / (1 << n)
    return bits, U, D


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("n,q,seed", [(1, 1, 0), (2, 1, 1), (3, 2, 2), (4, 2, 3), (4, 3, 4), (6, 1, 5), (7, 2, 6),
                                      (8, 3, 7), (9, 2, 8), (10, 3, 9), (10, 1, 10)])
def test_gate_vs_dense_definition(m, torch_cuda, dtype, n, q, seed):
    torch = torch_cuda
    bits, U, D = rand_case(n, q, seed)
    want = qgate.apply_gate_dense(D, U, bits)
    tdt = torch.complex128 if dtype == "c128" else torch.complex64
    rho = torch.from_numpy(D.astype(np.complex128)).to(tdt).cuda().contiguous()
    m.moa_qgate_apply(rho, n, bits, U)
    torch.cuda.synchronize()
    got = rho.cpu().numpy().astype(np.complex128)
    tol = 1e-12 if dtype == "c128" else 2e-6
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= tol
    if dtype == "c128":
        assert abs(np.trace(got) - np.trace(D)) < 1e-11                      # trace preserved
        assert np.max(np.abs(got - got.conj().T)) < 1e-12                    # Hermitian


def test_fig_qubits_paper_example(m, torch_cuda):
    # n = 4, gated bits 0 and 2 (xaxb, t = <0 2 1 3 4 6 5 7>): X (x) X on those bits
    torch = torch_cuda
    rng = np.random.default_rng(11)
    D = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    X = np.array([[0, 1], [1, 0]], np.complex128)
    U = np.kron(X, X)
    rho = torch.from_numpy(D).cuda()
    m.moa_qgate_apply(rho, 4, [0, 2], U)
    assert np.allclose(rho.cpu().numpy(), qgate.apply_gate_virtual(D, U, [0, 2]), atol=1e-14)


@pytest.mark.parametrize("n,bits,dtype", [(13, [0, 5, 12], "c128"), (14, [3, 7], "c128"), (14, [13], "c128"),
                                          (14, [3, 9], "c128"), (14, [3, 9], "c64"), (13, [2, 7, 12], "c64"),
                                          (14, [0], "c64")])
def test_large_sampled_blocks(m, torch_cuda, n, bits, dtype):
    # full-size launches (several row groups per CTA, the bank-model row stride)
    torch = torch_cuda
    rng = np.random.default_rng(n)
    q = len(bits)
    U, _ = np.linalg.qr(rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q)))
    N = 1 << n
    rho = torch.randn(N, N, dtype=torch.complex128 if dtype == "c128" else torch.complex64, device="cuda")
    D = rho.cpu().numpy().reshape(-1).astype(np.complex128)
    m.moa_qgate_apply(rho, n, bits, U)
    torch.cuda.synchronize()
    got = rho.cpu().numpy().reshape(-1).astype(np.complex128)
    tol = 1e-12 if dtype == "c128" else 5e-6
    t = qgate.gate_permutation(n, bits)
    Q = 1 << q

    def off(vr, vc):
        i_vec = [(vr >> (n - 1 - p)) & 1 for p in range(n)] + [(vc >> (n - 1 - p)) & 1 for p in range(n)]
        return qgate.permuted_offset(i_vec, t)
    for _ in range(20):
        r, c = (int(v) for v in rng.integers(0, N // Q, 2))
        offs = np.array([[off(r * Q + a, c * Q + b) for b in range(Q)] for a in range(Q)])
        B = D[offs]
        assert np.max(np.abs(got[offs] - U @ B @ U.conj().T)) < tol


@pytest.mark.parametrize("bits", [[0, 14], [3, 9, 14]])
def test_max_size_sampled_blocks(m, torch_cuda, bits):
    # n = 15 (the ABI's maximum): a 2^15 x 2^15 complex64 matrix (8 GiB); the
    # sampled blocks are gathered on the device before and after the gate
    torch = torch_cuda
    n, q = 15, len(bits)
    rng = np.random.default_rng(150 + q)
    U, _ = np.linalg.qr(rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q)))
    N, Q = 1 << n, 1 << q
    g = torch.Generator(device="cuda").manual_seed(15)
    rho = torch.randn(N, N, dtype=torch.complex64, device="cuda", generator=g)
    t = qgate.gate_permutation(n, bits)

    def off(vr, vc):
        i_vec = [(vr >> (n - 1 - p)) & 1 for p in range(n)] + [(vc >> (n - 1 - p)) & 1 for p in range(n)]
        return qgate.permuted_offset(i_vec, t)
    blocks = []
    for _ in range(16):
        r, c = (int(v) for v in rng.integers(0, N // Q, 2))
        blocks.append(np.array([[off(r * Q + a, c * Q + b) for b in range(Q)] for a in range(Q)]))
    blocks.append(np.array([[off((N // Q - 1) * Q + a, (N // Q - 1) * Q + b) for b in range(Q)] for a in range(Q)]))
    idx = torch.from_numpy(np.concatenate([b.reshape(-1) for b in blocks])).cuda()
    flat = rho.view(-1)
    before = flat[idx].cpu().numpy().astype(np.complex128)
    m.moa_qgate_apply(rho, n, bits, U)
    torch.cuda.synchronize()
    after = flat[idx].cpu().numpy().astype(np.complex128)
    for k in range(len(blocks)):
        B = before[k * Q * Q:(k + 1) * Q * Q].reshape(Q, Q)
        A = after[k * Q * Q:(k + 1) * Q * Q].reshape(Q, Q)
        assert np.max(np.abs(A - U @ B @ U.conj().T)) < 5e-6

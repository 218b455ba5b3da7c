"""Pins of the density-matrix gate oracle (oracle/qgate.py; PAPER.md Ch.6,
SURVEY §8(f) f4) against the paper's printed examples and the mathematics --
never against itself.  CPU only."""
import os

import numpy as np
import pytest

from oracle import qgate

HERE = os.path.dirname(os.path.abspath(__file__))


def _panel(name):
    rows, cur = {}, None
    for line in open(os.path.join(HERE, "golden", "qubits_fig.txt")):
        line = line.rstrip("\n")
        if line.startswith("#") or not line:
            continue
        if line in ("LEFT", "RIGHT"):
            cur = line
            continue
        if cur == name:
            r = int(line[:4], 2)
            cells = {}
            for k in range(16):
                c = line[6 + 3 * k:9 + 3 * k].strip()
                if c:
                    cells[k] = c
            rows[r] = cells
    return rows


def test_transpose_vectors_printed_in_the_paper():
    # bits 0,2 (xaxb) -> <0 2 1 3 4 6 5 7>; bits 1,2 (xabx) -> <0 3 1 2 4 7 5 6>
    assert qgate.gate_permutation(4, [0, 2]) == [0, 2, 1, 3, 4, 6, 5, 7]
    assert qgate.gate_permutation(4, [1, 2]) == [0, 3, 1, 2, 4, 7, 5, 6]
    assert qgate.gate_permutation(4, [0, 1]) == list(range(8))      # already low bits: identity
    with pytest.raises(ValueError):
        qgate.gate_permutation(4, [1, 1])
    with pytest.raises(ValueError):
        qgate.gate_permutation(4, [4])


def test_fig_qubits_right_layout_viewed_through_eq_generic_is_the_left_layout():
    # Fig. qubits: the scattered xaxb layout, read through
    # @D + gamma(i[t]; s) with t = <0 2 1 3 4 6 5 7>, is the block-diagonal xxab layout
    right, left = _panel("RIGHT"), _panel("LEFT")
    D = np.full((16, 16), "", dtype=object)
    for r, cells in right.items():
        for c, v in cells.items():
            D[r, c] = v
    V = qgate.block_view_matrix(D, [0, 2])
    for r in range(16):
        for c in range(16):
            assert V[r, c] == left[r].get(c, ""), (r, c)


@pytest.mark.parametrize("n,bits", [(4, [0, 2]), (4, [1, 2]), (5, [4, 1]), (5, [0, 3, 4])])
def test_view_of_a_gate_operator_is_block_diagonal(n, bits):
    # the purpose of t: in the view, an operator that
    # acts only on the gated bits couples indices within one 2^q block only --
    # pins the reading of i[t] (R15) for the non-involutive xabx vector
    rng = np.random.default_rng(3)
    q = len(bits)
    U, _ = np.linalg.qr(rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q)))
    V = qgate.block_view_matrix(qgate.full_unitary(n, U, bits), bits)
    Q = 1 << q
    for r in range(1 << (n - q)):
        for c in range(1 << (n - q)):
            blk = V[r * Q:(r + 1) * Q, c * Q:(c + 1) * Q]
            if r == c:
                assert np.allclose(blk, U)
            else:
                assert not blk.any()


def test_full_unitary_is_kron_for_the_lowest_bits_and_x_flips_a_basis_state():
    rng = np.random.default_rng(1)
    for n, q in [(3, 1), (4, 2), (5, 3)]:
        A = rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q))
        U, _ = np.linalg.qr(A)
        assert np.allclose(qgate.full_unitary(n, U, list(range(q))), np.kron(np.eye(1 << (n - q)), U))
    X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    rho0 = np.zeros((2, 2), np.complex128)
    rho0[0, 0] = 1
    out = qgate.apply_gate_virtual(rho0, X, [0])
    assert np.array_equal(out, np.array([[0, 0], [0, 1]], dtype=np.complex128))   # |0><0| -> |1><1|


@pytest.mark.parametrize("n,bits", [(2, [1]), (3, [0, 2]), (4, [1, 2]), (4, [0, 2]), (4, [3]), (5, [0, 2, 4]),
                                    (5, [1, 3, 4]), (5, [4, 3])])
def test_virtual_algorithm_equals_the_dense_definition(n, bits):
    rng = np.random.default_rng(10 + n)
    q = len(bits)
    A = rng.standard_normal((1 << q, 1 << q)) + 1j * rng.standard_normal((1 << q, 1 << q))
    U, _ = np.linalg.qr(A)
    M = rng.standard_normal((1 << n, 1 << n)) + 1j * rng.standard_normal((1 << n, 1 << n))
    D = M @ M.conj().T
    D /= np.trace(D)
    got = qgate.apply_gate_virtual(D, U, bits)
    want = qgate.apply_gate_dense(D, U, bits)
    assert np.max(np.abs(got - want)) < 1e-12
    assert abs(np.trace(got) - 1) < 1e-12                              # trace preserved
    assert np.max(np.abs(got - got.conj().T)) < 1e-12                  # Hermitian
    if q < n:                                                          # gates on disjoint bits commute
        other = [b for b in range(n) if b not in bits][:1]
        V2, _ = np.linalg.qr(rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2)))
        ab = qgate.apply_gate_dense(qgate.apply_gate_dense(D, U, bits), V2, other)
        ba = qgate.apply_gate_dense(qgate.apply_gate_dense(D, V2, other), U, bits)
        assert np.max(np.abs(ab - ba)) < 1e-12

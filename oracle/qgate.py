"""oracle/qgate.py -- TEST INFRASTRUCTURE ONLY: the density-matrix gate of
PAPER.md Ch.6, written from the paper, plain numpy / Python.

Only tests/ may import it; it shares no code with paper_0803_2386_b200/.

Conventions (PAPER.md Ch.6, "Assumptions in the Example"):
  * bits are numbered right to left (bit 0 least significant);
  * hypercube coordinate positions are numbered left to right, so position p
    of an n-bit half is bit n-1-p;
  * the 2^n x 2^n density matrix D is the 2n-cube D_h = <2n> rho-hat 2 rho-hat D
    (row bits first, then column bits);
  * a gate U on q qubits is indexed so that bit j of U's row / column index is
    the j-th LOWEST gated bit.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def gate_permutation(n: int, gated_bits: Sequence[int]) -> List[int]:
    """The transpose vector t of the 2n-cube that moves the gated bits to the
    diagonal (the worked rows "swap bits 1 and 2", "<0 2 1 3 4 6 5 7>
    is the transpose vector"): within each n-half the coordinate positions are
    stably partitioned, ungated positions first, gated last; the column half
    repeats the row half shifted by n."""
    gated = set(int(b) for b in gated_bits)
    if len(gated) != len(list(gated_bits)) or any(b < 0 or b >= n for b in gated):
        raise ValueError("gated bits must be distinct and in [0, n)")
    pos_gated = {n - 1 - b for b in gated}
    half = [p for p in range(n) if p not in pos_gated] + [p for p in range(n) if p in pos_gated]
    return half + [p + n for p in half]


def permuted_offset(i_vec: Sequence[int], t: Sequence[int]) -> int:
    """Eq. generic: i psi (t transpose D) = @D + gamma(i[t]; s),
    s = <2n> rho-hat 2.  Reading R15: coordinate k of the view is
    coordinate t[k] of the original, so the original index i[t] has component
    t[k] equal to i[k] -- the reading under which BOTH printed vectors move the
    gated bits to the diagonal (for the involutive xaxb vector every reading
    agrees; for xabx, <0 3 1 2 4 7 5 6>, only this one does)."""
    it = [0] * len(t)
    for k, tk in enumerate(t):
        it[tk] = i_vec[k]
    off = 0
    for bit in it:                       # gamma on an all-2 shape (Horner)
        off = off * 2 + int(bit)
    return off


def block_view_matrix(D: np.ndarray, gated_bits: Sequence[int]) -> np.ndarray:
    """The block-diagonalising view (t transpose D_h), materialised element by
    element through Eq. generic (for tests; the algorithm never builds it)."""
    N = D.shape[0]
    n = N.bit_length() - 1
    t = gate_permutation(n, gated_bits)
    rav = D.reshape(-1)
    V = np.empty_like(D)
    for vr in range(N):
        for vc in range(N):
            i_vec = [(vr >> (n - 1 - p)) & 1 for p in range(n)] + [(vc >> (n - 1 - p)) & 1 for p in range(n)]
            V[vr, vc] = rav[permuted_offset(i_vec, t)]
    return V


def apply_gate_virtual(D: np.ndarray, U: np.ndarray, gated_bits: Sequence[int]) -> np.ndarray:
    """The paper's algorithm: view D as 2^{n-q} x 2^{n-q}
    blocks of 2^q x 2^q through the permuted indexing, apply the gate to every
    block, B <- U B U^dagger, and write back -- no permutation matrices."""
    N = D.shape[0]
    n = N.bit_length() - 1
    q = len(gated_bits)
    Q = 1 << q
    V = block_view_matrix(D, gated_bits)
    for r in range(N // Q):
        for c in range(N // Q):
            B = V[r * Q:(r + 1) * Q, c * Q:(c + 1) * Q]
            V[r * Q:(r + 1) * Q, c * Q:(c + 1) * Q] = U @ B @ U.conj().T
    # scatter back through the same map
    t = gate_permutation(n, gated_bits)
    out = np.empty_like(D).reshape(-1)
    for vr in range(N):
        for vc in range(N):
            i_vec = [(vr >> (n - 1 - p)) & 1 for p in range(n)] + [(vc >> (n - 1 - p)) & 1 for p in range(n)]
            out[permuted_offset(i_vec, t)] = V[vr, vc]
    return out.reshape(N, N)


def full_unitary(n: int, U: np.ndarray, gated_bits: Sequence[int]) -> np.ndarray:
    """The textbook operator of a gate on a subset of qubits, written out:
    U_full[i, j] = U[g(i), g(j)] if i and j agree on every ungated bit, else 0,
    where g(x) packs the gated bits of x (lowest gated bit -> bit 0).
    Independent of the transpose vector."""
    N = 1 << n
    bits = sorted(int(b) for b in gated_bits)
    gmask = sum(1 << b for b in bits)

    def g(x):
        return sum(((x >> b) & 1) << j for j, b in enumerate(bits))

    Uf = np.zeros((N, N), dtype=np.complex128)
    for i in range(N):
        for j in range(N):
            if (i & ~gmask) == (j & ~gmask):
                Uf[i, j] = U[g(i), g(j)]
    return Uf


def apply_gate_dense(D: np.ndarray, U: np.ndarray, gated_bits: Sequence[int]) -> np.ndarray:
    """D <- U_full D U_full^dagger with dense matrices (the definition)."""
    n = D.shape[0].bit_length() - 1
    Uf = full_unitary(n, U, gated_bits)
    return Uf @ D @ Uf.conj().T

"""Pins of the C oracle (oracle/oracle.c) against what the paper and the
mathematics fix -- never against itself.  CPU only."""
import numpy as np
import pytest

import oracle
import synth
from conftest import golden_lines

RNG_SEED = 12345


def rand(n, seed=RNG_SEED):
    return synth.fill(n, seed, synth.UNIFORM)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# --- O1: P_n -------------------------------------------------------------------
def test_bitrev_hand_values():
    # SPEC.md S:290-292 (derived by reversing bit strings)
    assert list(oracle.bitrev_perm(2)) == [0, 1]
    assert list(oracle.bitrev_perm(4)) == [0, 2, 1, 3]
    assert list(oracle.bitrev_perm(8)) == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("t", range(0, 13))
def test_bitrev_involution_and_action(t):
    n = 1 << t
    p = oracle.bitrev_perm(n)
    assert np.array_equal(p[p], np.arange(n))           # P_n o P_n = id
    x = rand(n)
    y = oracle.bitrev(x)
    assert np.array_equal(y, x[p])                        # element i moves to bitrev(i)


def test_bitrev_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        oracle.bitrev_perm(12)


# --- O3: the definition -----------------------------------------------------------
def test_direct_dft_hand_cases():
    for ln in golden_lines("dft_hand.txt"):
        a, b = ln.split(":")
        xi = np.array([float(v) for v in a.split()]).view(np.complex128)
        xo = np.array([float(v) for v in b.split()]).view(np.complex128)
        assert np.allclose(oracle.dft_direct(xi), xo, atol=1e-15)
        if (xi.size & (xi.size - 1)) == 0:
            assert np.allclose(oracle.fft_radix2(xi), xo, atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 16, 64])
def test_direct_dft_vs_textbook_matrix(n):
    # brute force: the n x n DFT matrix written out with numpy's exp
    x = rand(n, 7)
    j = np.arange(n)
    F = np.exp(-2j * np.pi * np.outer(j, j) / n)
    assert rel_l2(oracle.dft_direct(x), F @ x) < 1e-14


def test_direct_dft_vs_numpy_fft():
    for n in [16, 256, 1024, 1000]:
        x = rand(n, 3)
        assert rel_l2(oracle.dft_direct(x), np.fft.fft(x)) < 1e-14


# --- O2: fftpsirad2 ----------------------------------------------------------------
@pytest.mark.parametrize("t", range(0, 11))
def test_radix2_vs_direct_dft(t):
    # BASELINE.json: the oracle is checked against the O(n^2) direct DFT on n <= 2^10
    n = 1 << t
    x = rand(n, 100 + t)
    assert rel_l2(oracle.fft_radix2(x), oracle.dft_direct(x)) < 1e-14


@pytest.mark.parametrize("t", [1, 4, 10, 16, 20])
def test_radix2_closed_forms(t):
    n = 1 << t
    eps = 10 * n * np.finfo(float).eps
    delta = np.zeros(n, np.complex128)
    delta[0] = 1
    assert np.max(np.abs(oracle.fft_radix2(delta) - 1)) < eps          # impulse -> all ones
    ones = np.ones(n, np.complex128)
    y = oracle.fft_radix2(ones)                                          # constant -> n delta
    assert abs(y[0] - n) < eps * n and np.max(np.abs(y[1:])) < eps * n
    # pure exponential e^{+2 pi i k0 j / n} -> n delta_{k,k0}; fixes the forward sign (reading R1)
    k0 = (3 * n) // 7 if n > 1 else 0
    j = np.arange(n)
    e = np.exp(2j * np.pi * ((k0 * j) % n) / n)
    y = oracle.fft_radix2(e)
    assert abs(y[k0] - n) < eps * n
    y[k0] = 0
    assert np.max(np.abs(y)) < eps * n


@pytest.mark.parametrize("t", [3, 12, 18])
def test_radix2_parseval_linearity_roundtrip(t):
    n = 1 << t
    x, y = rand(n, 1), rand(n, 2)
    X, Y = oracle.fft_radix2(x), oracle.fft_radix2(y)
    assert abs(np.vdot(X, X).real - n * np.vdot(x, x).real) < 1e-12 * n * np.vdot(x, x).real
    a, b = 0.37 - 1.2j, -2.5 + 0.25j
    assert rel_l2(oracle.fft_radix2(a * x + b * y), a * X + b * Y) < 1e-14
    back = np.conj(oracle.fft_radix2(np.conj(X))) / n                # inverse via conjugation
    assert rel_l2(back, x) < 1e-14


@pytest.mark.parametrize("t", [12, 16, 20])
def test_radix2_vs_numpy(t):
    n = 1 << t
    x = synth.fill(n, 9, synth.NORMAL)
    assert rel_l2(oracle.fft_radix2(x), np.fft.fft(x)) < 1e-14


def test_radix2_rows():
    n, b = 256, 5
    x = rand(n * b, 4)
    y = oracle.fft_radix2_rows(x, n)
    assert rel_l2(y.reshape(b, n), np.fft.fft(x.reshape(b, n), axis=1)) < 1e-14


# --- sampled bins (O3 restricted) ------------------------------------------------------
def test_dft_bins_vs_direct_all_bins():
    for n in [1, 2, 64, 1024]:
        x = rand(n, 5)
        ref = oracle.dft_direct(x)
        got = oracle.dft_bins(x, n, np.arange(n))
        assert rel_l2(got, ref) < 1e-15


def test_dft_bins_rows_and_c64():
    n, b = 1 << 14, 3
    x = rand(n * b, 6)
    rows = np.array([0, 2, 1, 2])
    bins = np.array([0, 77, n - 1, 5000])
    ref = np.fft.fft(x.reshape(b, n), axis=1)[rows, bins]
    assert np.max(np.abs(oracle.dft_bins(x, n, bins, rows) - ref)) < 1e-10
    x32 = x.astype(np.complex64)
    ref32 = np.fft.fft(x32.astype(np.complex128).reshape(b, n), axis=1)[rows, bins]
    assert np.max(np.abs(oracle.dft_bins(x32, n, bins, rows) - ref32)) < 1e-10


def test_dft3_bins_brute_force():
    for shape in [(8, 8, 8), (4, 8, 16), (1, 2, 4)]:
        N = int(np.prod(shape))
        x = synth.fill(N, 11, synth.NORMAL).reshape(shape)
        ref = np.fft.fftn(x)
        ks = np.array([(a, b, c) for a in range(shape[0]) for b in range(shape[1]) for c in range(shape[2])])
        got = oracle.dft3_bins(np.ascontiguousarray(x.reshape(-1)), shape, ks)
        assert rel_l2(got, ref.reshape(-1)) < 1e-14


# --- O4: the lifted (cache-optimized) FFT --------------------------------------------
def test_lifted_plan_paper_examples():
    for ln in golden_lines("weights_n32_c4.txt"):
        if ln.startswith("plan"):
            f = ln.split()
            n, c, lm, pm = int(f[1]), int(f[2]), int(f[5]), int(f[7])
            assert oracle.lifted_plan(n, c) == (lm, pm)


def test_lifted_plan_invariants():
    for t in range(1, 20):
        for lc in range(1, 22):
            lm, pm = oracle.lifted_plan(1 << t, 1 << lc)
            assert 1 <= pm <= lc and pm + lm * lc == t      # n = 2^{p_max} c^{l_max}
            if lc >= t:
                assert lm == 0                                  # c >= n: unblocked control


def _golden_rows(key):
    for ln in golden_lines("reshape_transpose_n32_c4.txt"):
        k, v = ln.split(":")
        if k.strip() == key:
            return [int(x) for x in v.replace("|", " ").split()]
    raise KeyError(key)


def test_reshape_transpose_paper_example():
    x = np.arange(32).astype(np.complex128)
    s1 = oracle.reshape_transpose(x, 4)
    assert [int(v.real) for v in s1] == _golden_rows("reshape3")
    s2 = oracle.reshape_transpose(s1, 4)
    assert [int(v.real) for v in s2] == _golden_rows("xdeqn")


def test_final_transpose_inverts_reshape_transposes():
    # F_{n, l_max log2 c} o S^{l_max} = id (reading R5), all n <= 2^12, all c
    for t in range(1, 13):
        n = 1 << t
        x = np.arange(n).astype(np.complex128)
        for lc in range(1, t + 2):
            lm, _ = oracle.lifted_plan(n, 1 << lc)
            y = x.copy()
            for _ in range(lm):
                y = oracle.reshape_transpose(y, 1 << lc) if (1 << lc) <= n else y
            z = oracle.final_transpose(y, lm * lc)
            assert np.array_equal(z, x), (n, lc)


@pytest.mark.parametrize("t", range(1, 11))
def test_lifted_fft_matches_dft_for_every_c(t):
    n = 1 << t
    x = rand(n, 200 + t)
    ref = oracle.dft_direct(x)
    for lc in range(1, t + 2):
        assert rel_l2(oracle.fft_lifted(x, 1 << lc), ref) < 1e-14, (n, 1 << lc)


def test_lifted_fft_large_vs_numpy():
    n = 1 << 16
    x = synth.fill(n, 21, synth.NORMAL)
    for c in [16, 256, 1 << 16]:
        assert rel_l2(oracle.fft_lifted(x, c), np.fft.fft(x)) < 1e-14


# --- O5: 3-D ---------------------------------------------------------------------------
def test_fft3d_vs_brute_force_and_numpy():
    for shape in [(8, 8, 8), (4, 8, 16), (2, 1, 4)]:
        N = int(np.prod(shape))
        x = synth.fill(N, 31, synth.NORMAL).reshape(shape)
        got = oracle.fft3d(x)
        ks = np.array([(a, b, c) for a in range(shape[0]) for b in range(shape[1]) for c in range(shape[2])])
        brute = oracle.dft3_bins(np.ascontiguousarray(x.reshape(-1)), shape, ks).reshape(shape)
        assert rel_l2(got, brute) < 1e-14
        assert rel_l2(got, np.fft.fftn(x)) < 1e-14


def test_fft3d_plane_wave():
    shape = (16, 8, 32)
    k = (5, 3, 17)
    j0, j1, j2 = np.meshgrid(*[np.arange(s) for s in shape], indexing="ij")
    x = np.exp(2j * np.pi * (j0 * k[0] / shape[0] + j1 * k[1] / shape[1] + j2 * k[2] / shape[2]))
    y = oracle.fft3d(x)
    N = int(np.prod(shape))
    assert abs(y[k] - N) < 1e-9
    y[k] = 0
    assert np.max(np.abs(y)) < 1e-9


# ---------------------------------------------------------------- the + sign (inverse) variant
@pytest.mark.parametrize("t", [0, 1, 5, 10])
def test_plus_sign_direct_vs_textbook_and_radix2(t):
    # the fragment's weight EXP(+2 pi i row/L) read literally: kernel e^{+2 pi i jk/n}
    n = 1 << t
    x = rand(n, 300 + t)
    j = np.arange(n)
    F = np.exp(2j * np.pi * (np.outer(j, j) % n) / n)                   # the written-out matrix
    assert rel_l2(oracle.dft_direct_sign(x, +1), F @ x) < 1e-13
    assert rel_l2(oracle.fft_radix2_sign(x, +1), oracle.dft_direct_sign(x, +1)) < 1e-14
    assert rel_l2(oracle.fft_radix2_sign(x, -1), oracle.fft_radix2(x)) == 0.0


@pytest.mark.parametrize("t", [1, 8, 16])
def test_plus_sign_closed_forms_and_roundtrip(t):
    n = 1 << t
    eps = 10 * n * np.finfo(float).eps
    # impulse at k0 -> e^{+2 pi i k0 j / n} (the inverse of the forward closed form)
    k0 = (5 * n) // 11
    d = np.zeros(n, np.complex128)
    d[k0] = 1
    j = np.arange(n)
    assert np.max(np.abs(oracle.fft_radix2_sign(d, +1) - np.exp(2j * np.pi * ((k0 * j) % n) / n))) < eps
    # forward then + sign returns n x (the unnormalised inverse), numpy.fft.ifft as third party
    x = rand(n, 400 + t)
    assert rel_l2(oracle.fft_radix2_sign(oracle.fft_radix2(x), +1), n * x) < 1e-14
    assert rel_l2(oracle.fft_radix2_sign(x, +1), n * np.fft.ifft(x)) < 1e-13
    rows = oracle.fft_radix2_rows_sign(np.concatenate([x, 2 * x]), n, +1)
    assert rel_l2(rows[n:], 2 * rows[:n]) < 1e-15


def test_plus_sign_3d():
    x = rand(4 * 8 * 16, 77).reshape(4, 8, 16)
    assert rel_l2(oracle.fft3d_sign(x, +1), 512 * np.fft.ifftn(x)) < 1e-13
    assert rel_l2(oracle.fft3d_sign(oracle.fft3d(x), +1), 512 * x) < 1e-14

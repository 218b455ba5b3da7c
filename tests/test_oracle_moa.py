"""Pins of the MoA / psi index oracle (oracle/moa.py) against the paper's printed
worked examples (tests/golden/) and exhaustive algebraic laws.  CPU only."""
import itertools

import numpy as np
import pytest

import oracle
from conftest import golden_lines
from oracle import moa


def A60():
    return moa.reshape((3, 5, 4), moa.iota(60))


def test_psi_paper_examples():
    A = A60()
    for ln in golden_lines("moa_psi_examples.txt"):
        head, val = ln.split(":")
        f = head.split()
        idx = [int(v) for v in f[1:]]
        if f[0] == "psi":
            assert moa.psi(idx, A).rav == [int(v) for v in val.split()]
        elif f[0] == "reduce":
            # <1 2> psi (2 take (Phi A)) = <1 2> psi A; Phi = reverse on axis 0
            phiA = moa.MoaArray(A.shape, sum((moa.psi([i], A).rav for i in reversed(range(3))), []))
            t2 = moa.MoaArray((2,) + A.shape[1:], phiA.rav[: 2 * 20])
            r = moa.psi(idx, t2)
            assert list(r.shape) == [int(v) for v in val.split()[1:]]
            # the paper's psi-reduction <1 2> psi Phi A = <2> psi (<3-1-1> psi A)
            assert r.rav == moa.psi([3 - 1 - 1, idx[1]], A).rav


def test_psi_empty_index_and_gamma_roundtrip():
    A = A60()
    assert moa.psi([], A).rav == A.rav                      # <> psi A = A
    assert moa.gamma([2, 1, 3], (3, 5, 4)) == 47
    for off in range(60):
        assert moa.gamma(moa.gamma_inv(off, (3, 5, 4)), (3, 5, 4)) == off
    with pytest.raises(IndexError):
        moa.gamma([3, 0, 0], (3, 5, 4))


def test_reshape_modulo_rule_and_pi_empty():
    assert moa.pi([]) == 1
    assert moa.reshape((7,), moa.iota(3)).rav == [0, 1, 2, 0, 1, 2, 0]
    assert moa.reshape((2,), moa.iota(5)).rav == [0, 1]


def test_vector_ops():
    v = [0, 1, 2, 3, 4]
    assert moa.rotate(2, v) == [2, 3, 4, 0, 1] and moa.rotate(-2, moa.rotate(2, v)) == v
    for k in range(6):
        assert moa.cat(moa.take(k, v), moa.drop(k, v)) == v
    assert moa.take(-1, v) == [4] and moa.drop(-1, v) == [0, 1, 2, 3]


def test_reshape_transpose_paper_example():
    rows = {}
    for ln in golden_lines("reshape_transpose_n32_c4.txt"):
        k, v = ln.split(":")
        rows[k.strip()] = [int(x) for x in v.replace("|", " ").split()]
    x = list(range(32))
    assert moa.reshape((8, 4), moa.iota(32)).rav == rows["reshape1"]
    assert moa.transpose(moa.reshape((8, 4), moa.iota(32))).rav == rows["reshape2"]
    s1 = moa.reshape_transpose(x, 8, 4)
    assert s1 == rows["reshape3"]
    assert moa.reshape_transpose(s1, 8, 4) == rows["xdeqn"]


def test_hypercube_rotation_paper_examples():
    A = moa.reshape((2, 2, 2, 2), moa.reshape((4, 4), moa.iota(16)))
    B = moa.reshape((2, 2, 2, 2), moa.reshape((4, 4), moa.transpose(moa.reshape((4, 4), moa.iota(16)))))
    for ln in golden_lines("hypercube_rotation.txt"):
        f = [s.split() for s in ln.split(":")]
        if f[0][0] == "rot4":
            p, q, val = [int(v) for v in f[0][1:]], [int(v) for v in f[1]], int(f[2][0])
            assert moa.rotate(2, p) == q
            assert moa.psi(p, B).rav[0] == moa.psi(q, A).rav[0] == val
        else:
            vec = [int(v) for v in f[1]]
            if f[0][1] == "q_of_p":
                assert moa.rotate(2, list(range(5))) == vec
            elif f[0][1] == "b_vs_a":
                assert moa.rotate(2, list(range(5))) == vec
                Ah = moa.hypercube(list(range(32)))
                Bh = moa.hypercube(moa.reshape_transpose(list(range(32)), 8, 4))
                assert moa.transpose(Ah, vec).rav == Bh.rav
            else:
                assert moa.rotate(-2, list(range(5))) == vec
                Ah = moa.hypercube(list(range(32)))
                Bh = moa.hypercube(moa.reshape_transpose(list(range(32)), 8, 4))
                assert moa.transpose(Bh, vec).rav == Ah.rav


@pytest.mark.parametrize("t", range(1, 11))
def test_rotation_law_and_final_transpose_exhaustive(t):
    # S^l(iota n)[m] = rotl_t(m, l log2 c) and F o S^{l_max} = id for every c (reading R5/R6)
    n = 1 << t
    x = list(range(n))
    for lc in range(1, t + 1):
        c = 1 << lc
        y = x
        l_max, _ = oracle.lifted_plan(n, c)
        for l in range(1, l_max + 1):
            y = moa.reshape_transpose(y, n // c, c)
            sh = (l * lc) % t
            assert y == [((m << sh) | (m >> (t - sh))) & (n - 1) for m in range(n)]
        assert moa.final_transpose(y, l_max * lc) == x
        # the MoA statement of F equals the paper's C loop (oracle.c)
        z = oracle.final_transpose(np.array(y, dtype=np.complex128), l_max * lc)
        assert [int(v.real) for v in z] == x


@pytest.mark.parametrize("t", range(0, 11))
def test_bit_reversal_is_hypercube_reversal(t):
    n = 1 << t
    assert moa.bit_reversal(list(range(n))) == list(oracle.bitrev_perm(n))


def test_tvec_table():
    for ln in golden_lines("tvec_l8.txt"):
        j, v = ln.split(":")
        assert moa.t_vec(8, int(j)) == [int(x) for x in v.split()]


@pytest.mark.parametrize("l", range(1, 9))
def test_hypercube_pairs_equal_radix2_pairs(l):
    for j in range(l):
        assert sorted(moa.hypercube_pairs(l, j)) == sorted(moa.radix2_pairs(l, j + 1))


def test_weight_layouts_paper_example():
    n, c = 32, 4
    for ln in golden_lines("weights_n32_c4.txt"):
        if not ln.startswith("stage"):
            continue
        head, blocks, diag = ln.split(":")
        _, l, p, L = head.split()
        l, p, L = int(l), int(p), int(L)
        sig = [int(v) for v in blocks.split()[1:]]
        ex = moa.weight_exponents(n, c, l, p)
        v = 1 << p
        assert L == v * c ** l
        per_block = [[e for (m, e) in ex if m // v == b] for b in range(n // v)]
        for b, s in enumerate(sig):
            want = [s + jj * c ** l for jj in range(v // 2)]
            assert per_block[b] == want
        if "sigma+4" in diag:
            assert all(pb[1] - pb[0] == 4 for pb in per_block)


def test_plan_accounting():
    for t in range(1, 12):
        for lc in range(1, t + 1):
            pl = moa.lifted_plan(1 << t, 1 << lc)
            assert (1 << pl["p_max"]) * (1 << lc) ** pl["l_max"] == 1 << t
            for st in pl["stages"]:
                assert st["v"] * st["d_v"] * st["S_v"] == 1 << t
            assert len(pl["stages"]) == t                               # every radix-2 stage once


def test_pct_example_and_contiguity():
    for ln in golden_lines("pct_example.txt"):
        f = ln.replace(":", " ").split()
        j = [int(f[1])]
        shape = [int(v) for v in f[3:6]]
        assert moa.pct(j, shape) == (int(f[7]), int(f[9]))
    for shape in [(4, 6, 7), (2, 3, 4, 5), (8,)]:
        A = moa.reshape(shape, moa.iota(moa.pi(shape)))
        for k in range(len(shape) + 1):
            for j in itertools.product(*[range(s) for s in shape[:k]]):
                start, length = moa.pct(list(j), shape)
                assert moa.psi(list(j), A).rav == list(range(start, start + length))


# --- the B200 plan's lifting maps, executed by plain numpy --------------------------------
def execute_maps(x, passes):
    y = x.astype(np.complex128).copy()
    for ps in passes:
        load, store, tw = np.array(ps["load"]), np.array(ps["store"]), np.array(ps["tw"])
        lines = y[load]                                        # [line][j]
        R = ps["R"]
        F = np.exp(-2j * np.pi * np.outer(np.arange(R), np.arange(R)) / R)
        out = lines @ F.T                                      # DFT_R of every line
        out = out * np.exp(-2j * np.pi * tw / ps["twN"])
        z = np.empty_like(y)
        z[store] = out
        y = z
    return y


@pytest.mark.parametrize("radices,batch", [([4, 8], 1), ([8, 8], 2), ([2, 4, 8], 1), ([4, 2, 2, 4], 3),
                                           ([16], 2), ([8, 4, 16], 1), ([2, 2], 1)])
def test_lift_pass_maps_compute_the_dft(radices, batch):
    n = moa.pi(radices)
    passes = moa.lift_pass_maps(radices, batch)
    x = synth_input(n * batch)
    got = execute_maps(x, passes)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


def synth_input(n):
    import synth
    return synth.fill(n, 77, synth.UNIFORM)


def test_lift_maps_are_the_paper_transposes():
    # pass-0 load order over lines = S_{r,c} (Eq. reshape3) with r = R_0, c = n/R_0;
    # for two equal factors the last store is the final transpose F_{n, log2 c}.
    for r, c in [(8, 4), (4, 8), (16, 16)]:
        n = r * c
        ps = moa.lift_pass_maps([r, c])
        flat = [a for line in ps[0]["load"] for a in line]
        assert flat == moa.reshape_transpose(list(range(n)), r, c)
        if r == c:
            last = ps[1]
            out = [0] * n
            for line_l, line_s in zip(last["load"], last["store"]):
                for a, b in zip(line_l, line_s):
                    out[b] = a
            assert out == moa.final_transpose(list(range(n)), moa.ilog2(c))


@pytest.mark.parametrize("radices,batch", [([4, 8], 1), ([8, 8], 2), ([2, 4, 8], 1), ([4, 2, 2, 4], 3),
                                           ([16], 2), ([8, 4, 16], 1), ([32, 2, 4], 2)])
def test_lift_line_maps_pointwise(radices, batch):
    # the pointwise form (gamma / transpose evaluated per element, used for the
    # config liftings up to 2^30) executes to the DFT on its own, and agrees line
    # by line with the materialised maps
    n = moa.pi(radices)
    P = len(radices)
    ref_maps = moa.lift_pass_maps(radices, batch)
    passes = []
    for p in range(P):
        Sp = moa.pi(radices[p + 1:])
        Bp = batch * n // (radices[p] * Sp)
        rows = [moa.lift_line_maps(radices, batch, p, (o, j)) for o in range(Bp) for j in range(Sp)]
        ps = dict(R=radices[p], load=[r["load"] for r in rows], store=[r["store"] for r in rows],
                  tw=[r["tw"] for r in rows], twN=rows[0]["twN"])
        assert ps["load"] == ref_maps[p]["load"] and ps["store"] == ref_maps[p]["store"]
        assert ps["tw"] == ref_maps[p]["tw"] and ps["twN"] == ref_maps[p]["twN"]
        passes.append(ps)
    x = synth_input(n * batch)
    got = execute_maps(x, passes)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13

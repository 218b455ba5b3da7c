"""oracle/moa.py -- TEST INFRASTRUCTURE ONLY: the MoA / psi-calculus index algebra.

Plain-Python (small-case) implementation of the Mathematics-of-Arrays operators
of PAPER.md Ch.2 and the index maps of Ch.3-5, materialised element by element
so a reader can check each against the paper.  It is the oracle for every
integer map the CUDA path's psi-index layer emits; it shares no code with
paper_0803_2386_b200/ and never imports it.

Conventions (PAPER.md line numbers, "P:a-b"):
  * arrays are {shape, ravel} in zero-origin row-major order;
  * gamma is the row-major layout function, Horner form x_j = x_{j-1} s_j + p_j
    (Def. gammadef);
  * psi with a full index selects a scalar, with a partial index a sub-array
    (P:843-896), <> psi A = A;
  * reshape uses the modulo rule ravel[k mod tau];
  * generalised transpose `perm (/) A`: (perm (/) A)[p] = A[q] with
    q_a = p_{perm[a]} -- the convention fixed by Eq. b_vs_a and the
    relation <i j k l m> psi B = <k l m i j> psi A;
  * k phi v rotates the vector v left by k (Eq. q_eq);
  * k take v / k drop v: first k (k<0: last -k) / all but those.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple


def pi(v: Sequence[int]) -> int:
    """pi v: product of the components; pi <> = 1."""
    r = 1
    for x in v:
        r *= int(x)
    return r


@dataclass
class MoaArray:
    shape: Tuple[int, ...]
    rav: List

    def __post_init__(self):
        self.shape = tuple(int(s) for s in self.shape)
        assert len(self.rav) == pi(self.shape), "ravel length must equal tau(shape)"


def iota(n: int) -> MoaArray:
    """iota n = <0 1 ... n-1> (Fig. moa)."""
    return MoaArray((n,), list(range(n)))


def gamma(idx: Sequence[int], shape: Sequence[int]) -> int:
    """Row-major offset of a full index, Horner recurrence (Def. gammadef)."""
    assert len(idx) == len(shape)
    x = 0
    for p, s in zip(idx, shape):
        if not (0 <= p < s):
            raise IndexError(f"index {tuple(idx)} outside shape {tuple(shape)}")
        x = x * s + p
    return x


def gamma_inv(off: int, shape: Sequence[int]) -> Tuple[int, ...]:
    """Offset -> full index (Fig. moa, 'Translates offsets into indices given a shape')."""
    if not (0 <= off < pi(shape)):
        raise IndexError("offset out of range")
    out = []
    for s in reversed(shape):
        out.append(off % s)
        off //= s
    return tuple(reversed(out))


def reshape(shape: Sequence[int], a: MoaArray) -> MoaArray:
    """shape rho-hat a, with the modulo rule rav[k mod tau(a)]."""
    t = pi(shape)
    if t and not a.rav:
        raise ValueError("cannot reshape an empty array to a non-empty shape")
    return MoaArray(tuple(shape), [a.rav[k % len(a.rav)] for k in range(t)])


def psi(idx: Sequence[int], a: MoaArray) -> MoaArray:
    """idx psi a: full index -> 0-d array; partial index -> sub-array."""
    k = len(idx)
    assert k <= len(a.shape)
    for p, s in zip(idx, a.shape):
        if not (0 <= p < s):
            raise IndexError("psi index out of bounds")
    rest = a.shape[k:]
    start = gamma(list(idx), a.shape[:k]) * pi(rest) if k else 0
    return MoaArray(rest, a.rav[start:start + pi(rest)])


def take(k: int, v: Sequence) -> list:
    v = list(v)
    return v[:k] if k >= 0 else v[len(v) + k:]


def drop(k: int, v: Sequence) -> list:
    v = list(v)
    return v[k:] if k >= 0 else v[:len(v) + k]


def cat(a: Sequence, b: Sequence) -> list:
    return list(a) + list(b)


def rotate(k: int, v: Sequence) -> list:
    """k phi v: cyclic left rotation by k (negative: right); Eq. q_eq P:3946-3952."""
    v = list(v)
    if not v:
        return v
    k %= len(v)
    return v[k:] + v[:k]


def transpose(a: MoaArray, perm: Sequence[int] | None = None) -> MoaArray:
    """perm (/) a; default perm reverses the axes (2-D: the ordinary transpose)."""
    d = len(a.shape)
    if perm is None:
        perm = list(range(d - 1, -1, -1))
    perm = list(perm)
    assert sorted(perm) == list(range(d))
    bshape = [0] * d
    for ax in range(d):
        bshape[perm[ax]] = a.shape[ax]
    out = []
    for off in range(pi(bshape)):
        p = gamma_inv(off, bshape)
        q = [p[perm[ax]] for ax in range(d)]
        out.append(a.rav[gamma(q, a.shape)])
    return MoaArray(tuple(bshape), out)


def rav(a: MoaArray) -> list:
    return list(a.rav)


def pct(j: Sequence[int], shape: Sequence[int]) -> Tuple[int, int]:
    """psi Correspondence Theorem (Eq. psi_corr):
    rav(j psi xi) = (rav xi)[gamma(j; (tau j) take rho xi) * pi((tau j) drop rho xi)
                              + iota(pi((tau j) drop rho xi))]  -> (start, length)."""
    k = len(j)
    length = pi(drop(k, shape))
    start = (gamma(list(j), take(k, shape)) if k else 0) * length
    return start, length


# ---------------------------------------------------------------------------
# Ch.3-4 maps on iota n (values of the result = source offsets)
# ---------------------------------------------------------------------------
def ilog2(n: int) -> int:
    t = n.bit_length() - 1
    if n < 1 or (1 << t) != n:
        raise ValueError("not a power of two")
    return t


def reshape_transpose(x: Sequence, r: int, c: int) -> list:
    """S_{r,c}: <r c> rho-hat ((/) (<r c> rho-hat x))  (Eq. reshape3)."""
    a = reshape((r, c), MoaArray((len(x),), list(x)))
    return rav(reshape((r, c), transpose(a)))


def hypercube(x: Sequence) -> MoaArray:
    """(<d> rho-hat 2) rho-hat x."""
    d = ilog2(len(x))
    return reshape([2] * d, MoaArray((len(x),), list(x)))


def final_transpose(x: Sequence, sigma: int) -> list:
    """xi = <n> rho-hat (((-sigma) phi (iota d)) (/) ((<d> rho-hat 2) rho-hat x))
    (Eq. xihyper); equals out[t 2^sigma + s] = x[s 2^{d-sigma} + t]."""
    d = ilog2(len(x))
    return rav(transpose(hypercube(x), rotate(-sigma, list(range(d)))))


def bit_reversal(x: Sequence) -> list:
    """P_n x as the full axis reversal of the hypercube view."""
    return rav(transpose(hypercube(x)))


def t_vec(l: int, j: int) -> list:
    """t_j = (((l-1)-j) take c) ++ ((-1) take c) ++ (j take (((l-1)-j) drop c)),
    c = iota l (Eq. tvec)."""
    c = list(range(l))
    return cat(cat(take((l - 1) - j, c), take(-1, c)), take(j, drop((l - 1) - j, c)))


def hypercube_pairs(l: int, j: int) -> list:
    """Stage-j pairs of the three-loop ONF (Eq. final_loops):
    f = 2^j, g = 2^{j+1}; for m < 2^{l-1-j}, n < 2^j: (m g + n, m g + f + n)."""
    f, g = 1 << j, 1 << (j + 1)
    return [(m * g + n, m * g + f + n) for m in range(1 << (l - 1 - j)) for n in range(f)]


def radix2_pairs(t: int, q: int) -> list:
    """Pairs (col'+row, col'+row+L/2) of stage q of Fig. fftpsirad2."""
    n, L = 1 << t, 1 << q
    return [(col + row, col + row + L // 2) for col in range(0, n, L) for row in range(L // 2)]


def lifted_plan(n: int, c: int) -> dict:
    """Stage accounting of P:2740-2853 with the l_max reading R6:
    l_max = floor((t-1)/log2 c), p_max = t - l_max log2 c; per stage
    L = 2^p c^l, v = 2^p, d_v = c^l, S_v = n/(v d_v), S_B = 2^{p_max} c^{l_max-l-1}."""
    t, lc = ilog2(n), ilog2(c)
    assert t >= 1 and lc >= 1
    l_max = (t - 1) // lc
    p_max = t - l_max * lc
    stages = []
    for l in range(l_max + 1):
        for p in range(1, (lc if l < l_max else p_max) + 1):
            v, dv = 1 << p, c ** l
            stages.append(dict(l=l, p=p, L=v * dv, v=v, d_v=dv, S_v=n // (v * dv),
                               S_B=(2 ** p_max) * c ** (l_max - l - 1) if l < l_max else None))
    return dict(t=t, logc=lc, l_max=l_max, p_max=p_max, stages=stages)


def weight_exponents(n: int, c: int, l: int, p: int) -> list:
    """Exponent of w_L applied to the pair whose top element sits at position m,
    listed for every top position m (ascending): sigma + j c^l with
    sigma = m >> (t - l log2 c), j = m mod 2^{p-1} (reading R7 of the
    block-type index of P:2625-2643, 2728-2733)."""
    t, lc = ilog2(n), ilog2(c)
    v = 1 << p
    out = []
    for b in range(0, n, v):
        for j in range(v // 2):
            m = b + j
            out.append((m, (m >> (t - l * lc)) + j * c ** l))
    return out


# ---------------------------------------------------------------------------
# The lifting maps the B200 plan uses, materialised with MoA.
# ---------------------------------------------------------------------------
def lift_pass_maps(radices: Sequence[int], batch: int = 1) -> list:
    """For the lifting n = R_0 R_1 ... R_{P-1} (rows of a batch stacked), return,
    per pass p, a dict with integer arrays indexed [line][k]:
      load[line][k]  : source offset of point k of the line,
      store[line][k] : destination offset of DFT output k of the line,
      tw[line][k]    : twiddle exponent e (multiply by w_N^e, N = 'twN'),
    materialised from MoA expressions, independent of the plan's strides:
      pass p < P-1 views iota(batch n) as A_p = <B_p R_p S_p> rho-hat iota, S_p =
      R_{p+1}...R_{P-1}; a line is (o, j) (o = rows above, j < S_p), its points
      are <o k j> psi A_p; results go back to the same offsets (the lifted,
      not yet re-ordered layout) times w_{R_p S_p}^{j k};
      the last pass reads the rows of <B R_{P-1}> rho-hat iota and stores to the
      natural order given by the axis-reversing transpose of
      <batch R_0 ... R_{P-1}> rho-hat iota (the digit reversal, the lifted final
      transpose F)."""
    radices = list(radices)
    P = len(radices)
    n = pi(radices)
    total = batch * n
    base = iota(total)
    passes = []
    for p in range(P):
        Rp = radices[p]
        Sp = pi(radices[p + 1:])
        Bp = total // (Rp * Sp)
        A = reshape((Bp, Rp, Sp), base)
        load, store, tw = [], [], []
        if p < P - 1:
            for o in range(Bp):
                for j in range(Sp):
                    row = [psi((o, k, j), A).rav[0] for k in range(Rp)]
                    load.append(row)
                    store.append(list(row))
                    tw.append([(j * k) % (Rp * Sp) for k in range(Rp)])
            passes.append(dict(R=Rp, load=load, store=store, tw=tw, twN=Rp * Sp))
        else:
            shape = [batch] + radices
            z = reshape(shape, base)
            # axis order of the natural output: batch stays slowest, frequency
            # digits reversed (k_{P-1} slowest ... k_0 fastest)
            perm = [0] + [P - ax + 1 for ax in range(1, P + 1)]
            T = transpose(z, perm)
            where = [0] * total
            for pos, src in enumerate(T.rav):
                where[src] = pos
            for o in range(Bp):
                row = [psi((o, k, 0), A).rav[0] for k in range(Rp)]
                load.append(row)
                store.append([where[s] for s in row])
                tw.append([0] * Rp)
            passes.append(dict(R=Rp, load=load, store=store, tw=tw, twN=1))
    return passes


def lift_line_maps(radices: Sequence[int], batch: int, p: int, line: Tuple[int, int]) -> dict:
    """One line of lift_pass_maps(radices, batch)[p] without materialising the
    array, so the config liftings (n up to 2^30) can be checked line by line.
    The same MoA definitions, applied pointwise:
      * <o k j> psi (s rho-hat iota N) = gamma(<o k j>; s) -- psi of a full index
        selects the ravel element at its gamma offset (Def. gammadef
        P:1000-1019), and the ravel of iota is the offset itself;
      * the last pass's store position of source s is the offset, in the
        axis-reversing transpose T of <batch R_0 ... R_{P-1}> rho-hat iota, of the
        element whose value is s: T[q] = z[q'] with q'_a = q_{perm[a]}
        (transpose() above, Eq. b_vs_a), so s = gamma(q'; shape) and its
        position is gamma(q; bshape) with q_{perm[a]} = q'_a.
    line = (o, j): o the rows above axis p, j < S_p (0 for the last pass).
    -> dict(R, load, store, tw, twN) with one row each."""
    radices = list(radices)
    P = len(radices)
    n = pi(radices)
    total = batch * n
    Rp, Sp = radices[p], pi(radices[p + 1:])
    Bp = total // (Rp * Sp)
    o, j = line
    load = [gamma((o, k, j), (Bp, Rp, Sp)) for k in range(Rp)]
    if p < P - 1:
        return dict(R=Rp, load=load, store=list(load), tw=[(j * k) % (Rp * Sp) for k in range(Rp)],
                    twN=Rp * Sp)
    shape = [batch] + radices
    d = len(shape)
    perm = [0] + [P - ax + 1 for ax in range(1, P + 1)]
    bshape = [0] * d
    for ax in range(d):
        bshape[perm[ax]] = shape[ax]
    store = []
    for s in load:
        qp = gamma_inv(s, shape)          # q' : the element's index in z
        q = [0] * d
        for ax in range(d):
            q[perm[ax]] = qp[ax]
        store.append(gamma(q, bshape))
    return dict(R=Rp, load=load, store=store, tw=[0] * Rp, twN=1)

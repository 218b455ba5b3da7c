"""The C-ABI library on the CPU: it loads, exports every symbol include/moa_fft.h
declares, rejects bad arguments before touching CUDA, and its psi-index layer
emits ONF descriptors that are bit-exact against the oracle's MoA-materialised
maps.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth
from oracle import moa
from onf import enumerate_lines, enumerate_pass, run_dist, run_plan

import paper_0803_2386_b200 as m

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "moa_fft.h")).read()
    declared = set(re.findall(r"^\s*(?:moa_status_t|const char \*|int64_t|int)\s*\*?\s*(moa_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(m.EXPORTS), declared ^ set(m.EXPORTS)
    so = ctypes.CDLL(m._SO)
    for name in declared:
        assert hasattr(so, name), name


@pytest.mark.parametrize("args,status", [
    ((0, 1, "c128", 1), m.MOA_EINVAL), ((12, 1, "c128", 1), m.MOA_EINVAL), ((-4, 1, "c128", 1), m.MOA_EINVAL),
    ((1024, 0, "c128", 1), m.MOA_EINVAL), ((1024, 1, "c128", 3), m.MOA_EINVAL),
    ((1024, 1, "c128", 16), m.MOA_EINVAL), ((1024, 2, "c128", 2), m.MOA_EUNSUPPORTED),
    ((8, 1, "c128", 4), m.MOA_EUNSUPPORTED), ((1024, 1, "c128", 2), m.MOA_EINVAL),
    ((1 << 40, 1, "c64", 1), m.MOA_EINVAL),
])
def test_plan_argument_errors(args, status):
    with pytest.raises(m.MoaError) as ei:
        m.moa_fft_plan(*args)
    assert ei.value.status == status
    assert m.moa_fft_last_error()


def test_other_argument_errors():
    h = ctypes.c_void_p()
    assert m.lib.moa_fft_plan(ctypes.byref(h), 1024, 1, 7, 1) == m.MOA_EINVAL       # unknown dtype
    assert m.lib.moa_fft_plan(None, 1024, 1, 1, 1) == m.MOA_EINVAL                    # null out
    assert m.lib.moa_fft_exec(None, None, None, None) == m.MOA_EINVAL                 # null plan
    with pytest.raises(m.MoaError):
        m.moa_fft_plan_3d(1024, 1000, 8)
    with pytest.raises(m.MoaError):
        m.moa_fft_plan_3d(8192, 8, 8)
    with pytest.raises(m.MoaError):
        m.moa_fft_plan_lift(64, 1, "c128", [4, 4])                                      # product != n
    with pytest.raises(m.MoaError):
        m.moa_psi_describe(64, 1, "c128", [8, 3, 3])
    assert m.lib.moa_fft_destroy(None) == m.MOA_OK
    # plan flags: unknown bits, lifted order on a 3-D plan
    assert m.lib.moa_fft_plan_ex(ctypes.byref(h), 1024, 1, 1, 1, 32) == m.MOA_EINVAL
    for bad in (m.MOA_FFT_HYPERCUBE | m.MOA_FFT_UNBLOCKED, m.MOA_FFT_HYPERCUBE | m.MOA_FFT_LIFTED_ORDER):
        assert m.lib.moa_fft_plan_ex(ctypes.byref(h), 1024, 1, 1, 1, bad) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_plan_ex(ctypes.byref(h), 1024, 1, 1, 2, m.MOA_FFT_HYPERCUBE) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_plan_3d_ex(ctypes.byref(h), 8, 8, 8, 1, 1, m.MOA_FFT_HYPERCUBE) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_plan_ex(ctypes.byref(h), 1024, 1, 1, 2, m.MOA_FFT_UNBLOCKED) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_plan_ex(ctypes.byref(h), 1024, 1, 1, 1,
                                 m.MOA_FFT_UNBLOCKED | m.MOA_FFT_LIFTED_ORDER) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_plan_3d_ex(ctypes.byref(h), 8, 8, 8, 1, 1, m.MOA_FFT_LIFTED_ORDER) == m.MOA_EUNSUPPORTED
    assert m.lib.moa_fft_output_index(None, None, 0) == m.MOA_EINVAL


def test_planner_liftings():
    assert m.moa_plan_radices(1 << 10) == [1 << 10]
    assert m.moa_plan_radices(1 << 16) == [256, 256]
    assert m.moa_plan_radices(1 << 28, 1, "c128") == [512, 512, 1024]        # radix-32 lines: 3 passes
    assert m.moa_plan_radices(1 << 26, 1, "c64") == [512, 256, 512]          # measured table (r3l_planner)
    assert m.moa_plan_radices(1 << 30, 1, "c64") == [1024, 1024, 1024]       # FP32x2 radix-32: 3 passes
    assert m.moa_plan_radices(1 << 20, 1, "c128") == [1024, 1024]
    assert m.moa_plan_radices(1 << 29, 1, "c128") == [512, 1024, 1024]       # contiguous 1024-point last pass
    r3 = m.moa_plan_radices(1 << 27, 1, "c128")                              # odd t: three passes
    assert np.prod(r3) == 1 << 27 and len(r3) == 3 and r3[-1] == 1024
    for dt in ("c128", "c64"):
        for t in range(13, 34):                                              # multi-pass: strided lines <= 2^10
            r = m.moa_plan_radices(1 << t, 1, dt)
            assert len(r) >= 2 and max(r[:-1]) <= 1024 and r[-1] <= 4096
    for t in range(0, 34):
        r = m.moa_plan_radices(1 << t)
        assert int(np.prod(r)) == 1 << t and all(x <= 4096 for x in r)


def test_bench_config_tiles():
    # the tile shapes the measurements chose (profiles/r1_s7_*):
    # cfg2 two 256-point passes, 16-line tiles (256-byte runs)
    d2 = m.moa_psi_describe(1 << 16, 1024, "c128")
    assert [(1 << d["logR"], d["W"], d["threads"]) for d in d2] == [(256, 16, 256), (256, 16, 256)]
    # cfg4: three 1024-point complex64 passes (radix 32 x 32 on the FP32x2 pipe);
    # 16-line tiles (128-byte runs) where the loads are >= 1 MiB apart and where
    # contiguous lines are stored transposed; 8 lines for the 8 KiB-strided middle
    # pass, whose lifted weights favour two CTAs per SM (profiles/r6d_lfw.jsonl)
    d4 = m.moa_psi_describe(1 << 30, 1, "c64")
    assert [1 << d["logR"] for d in d4] == [1024, 1024, 1024]
    assert [d["W"] for d in d4] == [16, 8, 16] and [d["threads"] for d in d4] == [512, 256, 512]
    # the four-factor lifting it replaced: the 32 MiB-strided first pass takes 32 lines
    d4b = m.moa_psi_describe(1 << 30, 1, "c64", [256, 128, 128, 256])
    assert d4b[0]["W"] == 32 and d4b[0]["threads"] == 512 and d4b[1]["W"] == 16
    # cfg5: complex128 1024-point lines take 32 points per thread (radix 32 x 32; 512-point lines too)
    for d in m.moa_psi_describe_3d(1024, 1024, 1024, "c128"):
        assert d["logR"] == 10 and d["W"] * 32 == d["threads"] and d["threads"] <= 256
    # complex64 1024-point lines too; a contiguous (point-fast both sides)
    # >= 1024-point line is one CTA of its own
    d = m.moa_psi_describe_3d(64, 64, 1024, "c64")[0]
    assert d["logR"] == 10 and d["lf_load"] == 0 and d["lf_store"] == 0 and d["W"] == 1 and d["threads"] == 32
    # lines of <= 256 points keep 16 points per thread
    d = m.moa_psi_describe(1 << 16, 4, "c64")[1]
    assert d["logR"] == 8 and d["threads"] == d["W"] * 16


def _as_dict(load, store, tw):
    return {tuple(a): (tuple(b), tuple(c)) for a, b, c in zip(load.tolist(), store.tolist(), tw.tolist())}


@pytest.mark.parametrize("radices,batch", [([4, 8], 1), ([8, 8], 2), ([2, 4, 8], 1), ([4, 2, 2, 4], 3), ([16], 2),
                                           ([8, 4, 16], 1), ([2, 2], 1), ([32, 16], 2), ([64], 1)])
def test_psi_descriptors_bit_exact_vs_oracle_maps(radices, batch):
    n = int(np.prod(radices))
    got = m.moa_psi_describe(n, batch, "c128", radices)
    ref = moa.lift_pass_maps(radices, batch)
    assert len(got) == len(ref)
    for d, r in zip(got, ref):
        assert d["R"] == r["R"]
        load, store, tw = enumerate_pass(d)
        mine = _as_dict(load, store, tw if d["twN"] > 1 else np.zeros_like(tw))
        theirs = _as_dict(np.array(r["load"]), np.array(r["store"]), np.array(r["tw"]))
        assert mine == theirs
        if d["twN"] > 1:
            assert d["twN"] == r["twN"]
        # every element is loaded once and stored once (a permutation per pass)
        assert sorted(load.ravel().tolist()) == list(range(n * batch))
        assert sorted(store.ravel().tolist()) == list(range(n * batch))


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_psi_descriptors_bit_exact_at_config_liftings(cfg):
    # the planner's own descriptors at BASELINE.json's full sizes (cfg2 256*256
    # x 1024 rows, cfg3 2^28, cfg4 2^30 complex64) against the MoA maps of the
    # same lifting, evaluated pointwise (moa.lift_line_maps) on sampled lines:
    # the first and last lines and 300 random ones per pass, every point of each
    c = synth.CONFIGS[cfg]
    n, batch, dtype = c["n"], c["batch"], c["dtype"]
    passes = m.moa_psi_describe(n, batch, dtype)
    radices = [d["R"] for d in passes]
    assert int(np.prod(radices)) == n
    rng = np.random.default_rng(11)
    for p, d in enumerate(passes):
        assert d["ring"] == 0
        nlines = int(np.prod(d["ext"]))
        lines = np.unique(np.concatenate([[0, 1, 2, nlines - 2, nlines - 1], rng.integers(0, nlines, 300)]))
        load, store, tw = enumerate_lines(d, lines)
        Sp = int(np.prod(radices[p + 1:]))
        seen = set()
        for i in range(lines.size):
            o, k0, j = moa.gamma_inv(int(load[i, 0]), (batch * n // (d["R"] * Sp), d["R"], Sp))
            assert k0 == 0
            ref = moa.lift_line_maps(radices, batch, p, (o, j))
            assert load[i].tolist() == ref["load"]
            assert store[i].tolist() == ref["store"]
            if d["twN"] > 1:
                assert d["twN"] == ref["twN"] and tw[i].tolist() == ref["tw"]
            else:
                assert ref["twN"] == 1 or all(e == 0 for e in ref["tw"])
            seen.add((o, j))
        assert len(seen) == lines.size            # distinct ONF lines are distinct MoA lines


@pytest.mark.parametrize("n,batch,dtype", [(1 << 12, 2, "c128"), (1 << 16, 1, "c128"), (1 << 13, 1, "c64"),
                                           (1 << 20, 1, "c128"), (1 << 21, 1, "c64")])
def test_planner_descriptors_compute_the_dft(n, batch, dtype):
    # executing the planner's own ONF with plain numpy reproduces the oracle's DFT
    passes = m.moa_psi_describe(n, batch, dtype)
    x = synth.fill(n * batch, 5, synth.UNIFORM)
    got = run_plan(passes, x)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    for d in passes:                                    # tiles are legal (sm_100: 1024 threads, 227 KiB smem per CTA)
        assert d["threads"] <= 1024 and d["smem_bytes"] <= 227 * 1024
        if d["ndig"]:
            assert d["ext"][0] % d["W"] == 0


@pytest.mark.parametrize("rot", ["0", "1", "2", "3"])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_psi_3d_layouts(monkeypatch, rot, dtype):
    # in-place axis passes (0), the two rotating-layout schedules (1: z,y,x;
    # 2: z,x,y -- every pass reads contiguous lines, stores transposed) and the
    # mixed one (3: z in place, then strided loads / plane-strided stores)
    monkeypatch.setenv("MOA_FFT_3D_ROT", rot)
    for shape in [(8, 4, 16), (2, 32, 4), (16, 32, 64), (64, 8, 2)]:
        passes = m.moa_psi_describe_3d(*shape, dtype=dtype)
        if rot == "3":
            assert passes[0]["lf_load"] == 0 and passes[0]["lf_store"] == 0 and passes[-1]["dst"] == 1
        elif rot != "0":
            assert all(d["lf_load"] == 0 for d in passes)          # contiguous loads only
            assert [d["dst"] for d in passes][-1] == 1
        x = synth.fill(int(np.prod(shape)), 7, synth.NORMAL)
        got = run_plan(passes, x).reshape(shape)
        ref = oracle.fft3d(x.reshape(shape))
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


def test_psi_3d_descriptors(monkeypatch):
    monkeypatch.setenv("MOA_FFT_FUSE", "1")
    monkeypatch.setenv("MOA_FFT_3D_ROT", "0")
    for shape in [(8, 4, 16), (16, 16, 16), (2, 32, 4), (64, 64, 64), (16, 32, 64)]:
        passes = m.moa_psi_describe_3d(*shape)
        if min(shape[1:]) >= 32 and shape[0] >= 8:
            assert [d["ring"] for d in passes] == [2, 1, 0]     # z+y fused through the L2 ring
        x = synth.fill(int(np.prod(shape)), 6, synth.NORMAL)
        got = run_plan(passes, x).reshape(shape)
        ref = oracle.fft3d(x.reshape(shape))
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_1d_schedule_host_simulation(monkeypatch, p, peer):
    # processor-level lifting: every rank's ONF + the all-to-all chunk maps reproduce
    # the DFT -- with every exchange in NCCL (peer 0), or with E2 and E3 fused into
    # the stores of the pass before them (NVLink peer stores) and E1 left in NCCL
    monkeypatch.setenv("MOA_FFT_PEER", peer)
    N = 1 << 12
    x = synth.fill(N, 8, synth.UNIFORM)
    sch = [m.moa_dist_describe(r, p, N, "c64") for r in range(p)]
    kinds = [s[0] for s in sch[0]["steps"]]
    if peer == "0":
        assert kinds.count("alltoall") == 3
    else:
        assert kinds.count("alltoall") == 1 and kinds.count("fused") == 2
        # a fused pass never stores into a buffer it (or any pass since the last
        # synchronisation) reads
        for i, s in enumerate(sch[0]["steps"]):
            if s[0] == "fused":
                assert sch[0]["passes"][s[1]]["src"] != s[2]
                assert sch[0]["steps"][i + 1][0] == "barrier"
    outs = run_dist(sch, np.split(x, p))
    ref = oracle.fft_radix2(x)
    got = np.concatenate(outs)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_1d_lifted_order_schedule(monkeypatch, p, peer):
    # MOA_FFT_LIFTED_ORDER: no third all-to-all, no unpack; rank g holds X[g + p k2]
    # at offset k2 -- the final transpose is never executed
    N = 1 << 12
    x = synth.fill(N, 9, synth.UNIFORM)
    monkeypatch.setenv("MOA_FFT_PEER", peer)
    sch = [m.moa_dist_describe(r, p, N, "c128", flags=m.MOA_FFT_LIFTED_ORDER) for r in range(p)]
    kinds = [s[0] for s in sch[0]["steps"]]
    assert kinds.count("alltoall") + kinds.count("fused") == 2
    outs = run_dist(sch, np.split(x, p))
    ref = oracle.fft_radix2(x)
    for g in range(p):
        want = ref[g::p]
        assert np.linalg.norm(outs[g] - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.parametrize("peer", ["0", "1"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_3d_schedule_host_simulation(monkeypatch, p, peer):
    monkeypatch.setenv("MOA_FFT_PEER", peer)
    shape = (16, 8, 4)
    x = synth.fill(int(np.prod(shape)), 9, synth.NORMAL).reshape(shape)
    sch = [m.moa_dist_describe(r, p, shape, "c128") for r in range(p)]
    kinds = [s[0] for s in sch[0]["steps"]]
    assert kinds.count("alltoall") + kinds.count("fused") == 1
    if peer == "1":      # no synchronisation earlier in the exec: a barrier precedes the fused y-pass
        assert kinds[kinds.index("fused") - 1] == "barrier"
    shards = [np.ascontiguousarray(s).reshape(-1) for s in np.split(x, p, axis=0)]
    outs = run_dist(sch, shards)
    ref = oracle.fft3d(x)
    n1l = shape[1] // p
    for r in range(p):
        want = ref[:, r * n1l:(r + 1) * n1l, :].reshape(-1)       # y-slab [k0][k1_loc][k2]
        assert np.linalg.norm(outs[r] - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.parametrize("radices,batch,dtype", [([32, 32, 32, 32], 1, "c128"), ([32, 32, 32, 32], 2, "c64")])
def test_lift4_fused_descriptors_compute_the_dft(monkeypatch, radices, batch, dtype):
    # four-factor lifting as two L2-staged pairs (two HBM round trips)
    monkeypatch.setenv("MOA_FFT_LIFT4", "1")
    n = int(np.prod(radices))
    passes = m.moa_psi_describe(n, batch, dtype, radices)
    assert [d["ring"] for d in passes] == [2, 1, 2, 1]
    x = synth.fill(n * batch, 16, synth.NORMAL)
    got = run_plan(passes, x)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    # the planner picks it for the large single transforms
    assert [d["ring"] for d in m.moa_psi_describe(1 << 28, 1, "c128")] == [2, 1, 2, 1]
    assert [d["ring"] for d in m.moa_psi_describe(1 << 30, 1, "c64")] == [2, 1, 2, 1]


def test_fused_pair_descriptors_compute_the_dft(monkeypatch):
    # the L2-staged pass pair (ring of row buffers, slots reused) still computes the DFT
    monkeypatch.setenv("MOA_FFT_FUSE", "1")
    n, batch = 1 << 10, 100
    passes = m.moa_psi_describe(n, batch, "c128", [32, 32])
    assert passes[0]["ring"] == 2 and passes[1]["ring"] == 1
    assert passes[0]["ring_groups"] == batch and passes[0]["ring_slots"] < batch
    x = synth.fill(n * batch, 15, synth.UNIFORM)
    got = run_plan(passes, x)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    # cfg2's plan is one fused launch
    p2 = m.moa_psi_describe(1 << 16, 1024, "c128")
    assert [d["ring"] for d in p2] == [2, 1]


@pytest.mark.parametrize("n,batch,dtype,C,C_default", [
    (1 << 16, 3, "c128", 16, 0), (1 << 14, 2, "c128", 16, 8), (1 << 16, 2, "c64", 16, 0),
    (1 << 13, 3, "c128", 8, 8), (1 << 15, 2, "c128", 16, 8), (1 << 14, 3, "c64", 16, 8), (1 << 13, 2, "c64", 8, 8)])
def test_cluster_pair_descriptors(monkeypatch, n, batch, dtype, C, C_default):
    """The cluster level (MOA_FFT_CLUSTER=1, kernels.cu cluster_kernel): every
    group's pass-A stores stay inside the group (they go to the cluster's
    shared memory, slice q >> log2(G/C)), pass-B tile c of a group reads exactly
    slice c (its own CTA's shared memory), and the pair computes the DFT."""
    monkeypatch.setenv("MOA_FFT_CLUSTER", "1")
    A, B = m.moa_psi_describe(n, batch, dtype)
    assert (A["ring"], B["ring"]) == (3, 4)
    G, CC = A["ring_G"], A["ring_slots"]
    assert G == n and CC == C and A["ring_groups"] == batch
    _, sa, _ = enumerate_pass(A)
    la = np.arange(sa.shape[0]) // (sa.shape[0] // batch)
    assert (sa // G == la[:, None]).all()
    assert np.array_equal(np.sort(sa.ravel()), np.arange(n * batch))
    lb, _, _ = enumerate_pass(B)
    tile = np.arange(lb.shape[0]) // B["W"]
    assert ((lb % G) // (G // CC) == (tile % CC)[:, None]).all()
    assert (lb // G == (tile // CC)[:, None]).all()
    x = synth.fill(n * batch, 17, synth.UNIFORM)
    got = run_plan([A, B], x)
    ref = oracle.fft_radix2_rows(x, n)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    monkeypatch.delenv("MOA_FFT_CLUSTER")  # default: clusters of <= 8 CTAs of <= 256 threads
    dd = m.moa_psi_describe(n, batch, dtype)
    assert [d["ring"] for d in dd] == ([3, 4] if C_default else [0, 0])
    if C_default:
        assert dd[0]["ring_slots"] == C_default and dd[0]["threads"] == dd[1]["threads"] <= 256
    monkeypatch.setenv("MOA_FFT_CLUSTER", "0")
    assert [d["ring"] for d in m.moa_psi_describe(n, batch, dtype)] == [0, 0]


# ---------------------------------------------------------------- Ch.6 density-matrix gate (host side)
def test_qgate_transpose_vector_and_view_offsets_bit_exact_vs_oracle():
    from oracle import qgate
    assert m.moa_qgate_permutation(4, [0, 2]) == [0, 2, 1, 3, 4, 6, 5, 7]
    assert m.moa_qgate_permutation(4, [1, 2]) == [0, 3, 1, 2, 4, 7, 5, 6]
    rng = np.random.default_rng(4)
    for n in range(1, 8):
        for _ in range(4):
            q = int(rng.integers(1, min(3, n) + 1))
            bits = [int(b) for b in rng.choice(n, q, replace=False)]
            t = m.moa_qgate_permutation(n, bits)
            assert t == qgate.gate_permutation(n, bits)
            N = 1 << n
            for vr in range(N):
                for vc in range(N):
                    i_vec = [(vr >> (n - 1 - p)) & 1 for p in range(n)] + [(vc >> (n - 1 - p)) & 1 for p in range(n)]
                    assert m.moa_qgate_view_offset(n, bits, vr, vc) == qgate.permuted_offset(i_vec, t)
    for bad in [(4, [4]), (4, [1, 1]), (0, [0]), (4, [0, 1, 2, 3])]:
        with pytest.raises(m.MoaError):
            m.moa_qgate_permutation(*bad)

"""Test-side evaluation of the psi-layer's ONF descriptors, straight from the
semantics documented in include/moa_fft.h (loops over the line digits, affine
load / store addresses, twiddle exponent), plus a plain numpy executor of a
pass list / distributed schedule.  Used only by tests."""
import numpy as np


def enumerate_pass(d):
    """-> (load[line][k], store[line][k], tw_exp[line][k]) as int64 arrays, lines
    in ONF order (digit 0 fastest)."""
    R = d["R"]
    ext = d["ext"]
    nlines = int(np.prod(ext)) if ext else 1
    line = np.arange(nlines, dtype=np.int64)
    io = np.zeros(nlines, np.int64)
    oo = np.zeros(nlines, np.int64)
    te = np.zeros(nlines, np.int64)
    rest = line.copy()
    dig = np.zeros(nlines, np.int64)
    for e, si, so, st in zip(ext, d["in_str"], d["out_str"], d["tw_str"]):
        dig = rest % e
        rest //= e
        io += dig * si
        oo += dig * so
        te += dig * st
    if d.get("ring", 0) in (1, 2):
        # the slowest line bits are the group; on the ring side it addresses slot (g mod slots)
        grp = line // (nlines // d["ring_groups"])
        slot = (grp & (d["ring_slots"] - 1)) * d["ring_G"]
        if d["ring"] == 1:
            io += slot
        else:
            oo += slot
    k = np.arange(R, dtype=np.int64)
    load = io[:, None] + k[None, :] * d["in_kstr"]
    if d["out_ksplit"] < d["logR"]:
        lo = k & ((1 << d["out_ksplit"]) - 1)
        hi = k >> d["out_ksplit"]
        koff = lo * d["out_kstr"] + hi * d["out_kstr_hi"]
    else:
        koff = k * d["out_kstr"]
    store = oo[:, None] + koff[None, :]
    if d["twN"] > 1:
        tw = ((te[:, None] + d["tw_off"]) * k[None, :]) % d["twN"]
    else:
        tw = np.zeros_like(load)
    return load, store, tw


def group_of_lines(d):
    ext = d["ext"]
    nlines = int(np.prod(ext)) if ext else 1
    return np.arange(nlines) // (nlines // d["ring_groups"])


def run_pass(d, src, dst, lines_sel=None, enum=None):
    load, store, tw = enumerate_pass(d) if enum is None else enum
    if lines_sel is not None:
        load, store, tw = load[lines_sel], store[lines_sel], tw[lines_sel]
    R = d["R"]
    lines = src[load]
    if not d["kind"]:
        F = np.exp(-2j * np.pi * np.outer(np.arange(R), np.arange(R)) / R)
        lines = lines @ F.T
    if d["twN"] > 1:
        lines = lines * np.exp(-2j * np.pi * tw / d["twN"])
    dst[store] = lines


def run_plan(passes, x):
    bufs = {0: x.astype(np.complex128).copy(), 1: np.zeros(x.size, np.complex128),
            2: np.zeros(x.size, np.complex128), 3: np.zeros(x.size, np.complex128)}
    i = 0
    while i < len(passes):
        d = passes[i]
        if d.get("ring", 0) == 2:
            # fused pair: group by group through a ring of `slots` buffers (slot reuse exercised)
            B = passes[i + 1]
            ring = np.full(d["ring_slots"] * d["ring_G"], np.nan + 0j)
            ea, eb = enumerate_pass(d), enumerate_pass(B)
            la, lb = len(ea[0]) // d["ring_groups"], len(eb[0]) // B["ring_groups"]
            for g in range(d["ring_groups"]):          # lines of a group are contiguous in ONF order
                run_pass(d, bufs[d["src"]], ring, slice(g * la, (g + 1) * la), ea)
                run_pass(B, ring, bufs[B["dst"]], slice(g * lb, (g + 1) * lb), eb)
            i += 2
            continue
        if d.get("ring", 0) == 3:
            # cluster pair: A's stores land in the cluster's shared memory at their
            # group positions (the descriptors keep the plain layout), B reads them
            B = passes[i + 1]
            tmp = np.full(x.size, np.nan + 0j)
            run_pass(d, bufs[d["src"]], tmp)
            run_pass(B, tmp, bufs[B["dst"]])
            i += 2
            continue
        run_pass(d, bufs[d["src"]], bufs[d["dst"]])
        i += 1
    return bufs[1]


def run_dist(schedules, shards):
    """schedules[r] = moa_dist_describe(r, p, ...); shards[r] = rank r's input."""
    p = len(schedules)
    m = shards[0].size
    bufs = [{0: s.astype(np.complex128).copy(), 1: np.zeros(m, np.complex128), 2: np.zeros(m, np.complex128),
             3: np.zeros(m, np.complex128)} for s in shards]
    nsteps = len(schedules[0]["steps"])
    for i in range(nsteps):
        st = schedules[0]["steps"][i]
        if st[0] == "pass":
            for r in range(p):
                d = schedules[r]["passes"][schedules[r]["steps"][i][1]]
                run_pass(d, bufs[r][d["src"]], bufs[r][d["dst"]])
        elif st[0] == "barrier":
            continue
        elif st[0] == "fused":
            # the pass's stores, in its send layout, land in rank h's buffer t at g c
            _, _, t, c = st
            sends = []
            for r in range(p):
                d = schedules[r]["passes"][schedules[r]["steps"][i][1]]
                send = np.full(m, np.nan + 0j)
                run_pass(d, bufs[r][d["src"]], send)
                sends.append(send)
            for h in range(p):
                for g in range(p):
                    bufs[h][t][g * c:(g + 1) * c] = sends[g][h * c:(h + 1) * c]
        else:
            _, s, t, c = st
            snap = [bufs[g][s].copy() for g in range(p)]
            for h in range(p):
                for g in range(p):
                    bufs[h][t][g * c:(g + 1) * c] = snap[g][h * c:(h + 1) * c]
    return [b[1] for b in bufs]


def enumerate_lines(d, lines):
    """enumerate_pass restricted to the given ONF line numbers (large passes)."""
    R = d["R"]
    rest = np.asarray(lines, dtype=np.int64).copy()
    io = np.zeros(rest.size, np.int64)
    oo = np.zeros(rest.size, np.int64)
    te = np.zeros(rest.size, np.int64)
    for e, si, so, st in zip(d["ext"], d["in_str"], d["out_str"], d["tw_str"]):
        dig = rest % e
        rest //= e
        io += dig * si
        oo += dig * so
        te += dig * st
    k = np.arange(R, dtype=np.int64)
    load = io[:, None] + k[None, :] * d["in_kstr"]
    if d["out_ksplit"] < d["logR"]:
        koff = (k & ((1 << d["out_ksplit"]) - 1)) * d["out_kstr"] + (k >> d["out_ksplit"]) * d["out_kstr_hi"]
    else:
        koff = k * d["out_kstr"]
    store = oo[:, None] + koff[None, :]
    tw = ((te[:, None] + d["tw_off"]) * k[None, :]) % d["twN"] if d["twN"] > 1 else np.zeros_like(load)
    return load, store, tw

"""The processor-level lifting (step a8) across real processes: world_size-2
torch.distributed gloo ranks on the CPU.  Each rank takes its own schedule from
the C-ABI's psi-layer (moa_dist_describe), runs its local passes with the
test-side ONF executor and exchanges chunks with dist.all_to_all exactly as the
NCCL path does; the gathered result must equal the oracle's DFT."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _alltoall(buf_src, c, world):
    # ncclAlltoAll semantics: chunk h (c elements) of the send buffer goes to rank h,
    # chunk g of the receive buffer comes from rank g
    send = torch.from_numpy(np.ascontiguousarray(buf_src[:c * world]).view(np.float64).copy())
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    out = np.zeros(buf_src.size, np.complex128)
    out[:c * world] = recv.numpy().view(np.complex128)
    return out


def _worker(rank, world, port, kind, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_0803_2386_b200 as m
        from onf import run_pass

        if kind == "1d":
            N = 1 << 12
            x = synth.fill(N, 8, synth.UNIFORM)
            shard = x[rank * N // world:(rank + 1) * N // world]
            sch = m.moa_dist_describe(rank, world, N, "c128")
        else:
            shape = (16, 8, 32)
            x = synth.fill(int(np.prod(shape)), 9, synth.NORMAL).reshape(shape)
            shard = np.ascontiguousarray(np.split(x, world, axis=0)[rank]).reshape(-1)
            sch = m.moa_dist_describe(rank, world, shape, "c128")
        L = shard.size
        bufs = {0: shard.astype(np.complex128).copy(), 1: np.zeros(L, np.complex128),
                2: np.zeros(L, np.complex128), 3: np.zeros(L, np.complex128)}
        for st in sch["steps"]:
            if st[0] == "pass":
                d = sch["passes"][st[1]]
                run_pass(d, bufs[d["src"]], bufs[d["dst"]])
            elif st[0] == "barrier":
                dist.barrier()
            elif st[0] == "fused":                              # pass + all-to-all by its stores
                d = sch["passes"][st[1]]
                send = np.zeros(L, np.complex128)
                run_pass(d, bufs[d["src"]], send)
                bufs[st[2]] = _alltoall(send, st[3], world)
            else:
                _, s, t, c = st
                bufs[t] = _alltoall(bufs[s], c, world)
        out = [torch.empty(L * 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(bufs[1].view(np.float64).copy()))
        if rank == 0:
            q.put([o.numpy().view(np.complex128) for o in out])
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["1d", "3d"])
def test_processor_lifting_gloo_world2(kind):
    import oracle
    import synth

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = q.get(timeout=180)
    finally:
        for p in procs:
            p.join(5)
            if p.is_alive():
                p.kill()
    assert not isinstance(res, str), res
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    if kind == "1d":
        N = 1 << 12
        ref = oracle.fft_radix2(synth.fill(N, 8, synth.UNIFORM))
        got = np.concatenate(res)                              # natural blocks X[gM, (g+1)M)
    else:
        shape = (16, 8, 32)
        ref_full = oracle.fft3d(synth.fill(int(np.prod(shape)), 9, synth.NORMAL).reshape(shape))
        n1l = shape[1] // world                                # y-slab output [k0][k1_loc][k2]
        ref = np.concatenate([ref_full[:, r * n1l:(r + 1) * n1l, :].reshape(-1) for r in range(world)])
        got = np.concatenate(res)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12

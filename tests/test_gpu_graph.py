"""CUDA-graph capture of moa_fft_exec (the launch-bound inner loop captured
once and replayed -- the B200 way to run a fixed transform repeatedly).

Every plan kind must replay correctly: plain passes, the L2-staged pass pair
(its completion counters are reset on the stream inside the captured work,
ADVICE r1), the cluster pair, 3-D plans and the inverse.  Each replay runs on
new input contents and must be bit-identical to a direct exec of that input."""
import os

import numpy as np
import pytest

import synth

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


def make_plan(m, kind):
    env = {"fused": ("MOA_FFT_FUSE", "1"), "cluster": ("MOA_FFT_CLUSTER", "1")}.get(kind)
    old = os.environ.get(env[0]) if env else None
    if env:
        os.environ[env[0]] = env[1]
    try:
        if kind == "3d":
            return m.FFTPlan.plan_3d(32, 64, 128, dtype="c128")
        if kind == "3d_c64":
            return m.FFTPlan.plan_3d(64, 32, 64, dtype="c64")
        if kind == "inverse":
            return m.FFTPlan(1 << 14, 4, "c128", inverse=True, normalize=True)
        if kind == "three_pass":
            return m.FFTPlan(1 << 20, 2, "c64", radices=[64, 128, 128])
        return m.FFTPlan(1 << 16, 16, "c128")
    finally:
        if env:
            if old is None:
                del os.environ[env[0]]
            else:
                os.environ[env[0]] = old


@pytest.mark.parametrize("kind", ["plain", "fused", "cluster", "3d", "3d_c64", "inverse", "three_pass"])
def test_exec_graph_replay(m, torch_cuda, kind):
    torch = torch_cuda
    plan = make_plan(m, kind)
    if kind == "fused":
        assert [d["ring"] for d in plan.describe()][:2] == [2, 1]
    if kind == "cluster":
        assert [d["ring"] for d in plan.describe()] == [3, 4]
    c64 = kind in ("3d_c64", "three_pass")
    dt = torch.complex64 if c64 else torch.complex128
    n = plan.local_elems
    xs = [torch.from_numpy(synth.fill(n, 90 + i, synth.UNIFORM, "c64" if c64 else "c128")).cuda() for i in range(3)]
    want = [plan.exec(x).clone() for x in xs]
    x_static = torch.empty(n, dtype=dt, device="cuda")
    y_static = torch.empty(n, dtype=dt, device="cuda")
    x_static.copy_(xs[0])
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up on the capture stream
        plan.exec(x_static, y_static, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        plan.exec(x_static, y_static, stream=side)
    for rep in range(2):
        for i, x in enumerate(xs):
            x_static.copy_(x)
            g.replay()
            torch.cuda.synchronize()
            got = y_static.cpu().numpy()
            assert np.array_equal(got.view(np.uint8), want[i].cpu().numpy().view(np.uint8)), \
                f"{kind}: replay {rep} of input {i} differs from a direct exec"

"""The boundary from plain C (examples/c_example.c): include/moa_fft.h compiles
as C99 and a C program links libmoafft.so directly -- no Python, no torch.
Host part on CPU (planner / ψ-layer introspection, the Ch.6 transpose vector of
P:6409-6418, an argument error); the GPU part (impulse -> all ones, exec_host
round trip) under -m gpu."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    so_dir = os.path.join(ROOT, "paper_0803_2386_b200")
    if not os.path.exists(os.path.join(so_dir, "libmoafft.so")):
        pytest.skip("libmoafft.so not built")
    out = str(tmp_path_factory.mktemp("cex") / "c_example")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", f"-I{CUDA}/include",
           os.path.join(ROOT, "examples", "c_example.c"), f"-L{so_dir}", "-lmoafft", f"-L{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{so_dir}", f"-Wl,-rpath,{CUDA}/lib64", "-lm", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_c_example_host(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "qgate t: 0 2 1 3 4 6 5 7" in r.stdout          # the paper's printed transpose vector
    assert "radices 2^16 x 1024 c128: 256 256" in r.stdout
    assert "plan(n=3): status 1" in r.stdout                 # MOA_EINVAL before any allocation
    assert r.stdout.strip().endswith("OK")


@pytest.mark.gpu
def test_c_example_gpu(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "impulse 2^10" in r.stdout and r.stdout.strip().endswith("OK")

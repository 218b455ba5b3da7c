"""The NCCL bootstrap of the processor-level lifting (a8; include/moa_fft.h:
moa_fft_get_unique_id / moa_fft_dist_init) binds a usable libnccl in a process
that has not imported torch: the bundled NCCL (ncclAlltoAll) by default, an
older one (the system 2.27: grouped ncclSend / ncclRecv) when that is all there
is.  Each case in its own process: the C side binds one library per process."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SYS_NCCL = "/usr/lib/x86_64-linux-gnu/libnccl.so.2"

PROG = r"""
import sys
import paper_0803_2386_b200 as m
assert "torch" not in sys.modules
u = m.moa_fft_get_unique_id()
assert len(u) == 128 and any(u)
assert m.moa_fft_get_unique_id() != u          # a fresh id per call: the library is live
for rank, ngpu in ((0, 1), (0, 3), (2, 2), (-1, 4)):
    try:
        m.moa_fft_dist_init(rank, ngpu, u)
    except m.MoaError as e:
        assert "MOA_EINVAL" in str(e), e
    else:
        raise SystemExit(f"dist_init({rank}, {ngpu}) accepted")
m.moa_fft_dist_finalize()
print("ok")
"""


def _run(env_extra):
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("MOA_NCCL_LIB", None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", PROG], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_unique_id_default_library():
    _run({})


@pytest.mark.skipif(not os.path.exists(SYS_NCCL), reason="no system libnccl")
def test_unique_id_older_library_send_recv_fallback():
    _run({"MOA_NCCL_LIB": SYS_NCCL})


def test_unloadable_library_is_an_error_not_a_crash():
    env = dict(os.environ, PYTHONPATH=ROOT, MOA_NCCL_LIB="/nonexistent/libnccl.so.2", LD_LIBRARY_PATH="")
    prog = ("import paper_0803_2386_b200 as m\n"
            "try:\n    m.moa_fft_get_unique_id()\n"
            "except m.MoaError as e:\n    print('err', e)\nelse:\n    print('loaded')\n")
    r = subprocess.run([sys.executable, "-c", prog], env=env, capture_output=True, text=True, timeout=120)
    # either the search path still finds a libnccl (fine) or the call fails with MOA_ENCCL
    assert r.returncode == 0 and ("loaded" in r.stdout or "MOA_ENCCL" in r.stdout), r.stdout + r.stderr

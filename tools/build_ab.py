#!/usr/bin/env python3
"""Build an A/B variant of libmoafft.so whose kernels.cu comes from a git
revision or a file (the other objects from the working tree), for same-box timing
against the current build:  build_ab.py REV [NAME]  ->
paper_0803_2386_b200/build/ab/libmoafft_NAME.so; select it with
MOA_FFT_LIB_AB=paper_0803_2386_b200/build/ab/libmoafft_NAME.so."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402

spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_0803_2386_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
rev = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "prev"
out = os.path.join(b.BUILD, "ab")
os.makedirs(out, exist_ok=True)
src = os.path.join(out, f"_ab_{name}_kernels.cu")
with open(src, "w") as f:
    if os.path.exists(rev):  # a file path instead of a git revision
        f.write(open(rev).read())
    else:
        f.write(subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:paper_0803_2386_b200/csrc/kernels.cu"],
                                        text=True))
try:
    obj = os.path.join(out, f"kernels_{name}.o")
    subprocess.check_call([b.NVCC] + b._flags() + ["-I" + b.CSRC, "-c", src, "-o", obj])
    b.build()
    objs = [os.path.join(b.BUILD, f) for f in ("abi.cpp.o", "comm.cpp.o", "psi.cpp.o", "qgate.cu.o")] + [obj]
    so = os.path.join(out, f"libmoafft_{name}.so")
    subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", so] + objs + ["-ldl"])
    print(os.path.relpath(so, ROOT))
finally:
    os.remove(src)

"""Seeded synthetic inputs; see synth.c for the recipe.

Shared input generator for both sides of every parity check: it holds none of
the FFT's arithmetic.  `fill(...)` returns a numpy complex array of the global
elements [e0, e0+count) of a config's input.

Config recipes (BASELINE.json `configs`):
  cfg1: n=2^10,            c128, uniform[-1,1), seed 0
  cfg2: n=2^16 x 1024 rows, c128, uniform,       seed 1
  cfg3: n=2^28,            c128, standard normal, seed 2
  cfg4: n=2^30,            c64,  uniform,       seed 3
  cfg5: 1024^3 (3-D),      c128, standard normal, seed 4
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None

UNIFORM, NORMAL = 0, 1

CONFIGS = {
    "cfg1": dict(n=1 << 10, batch=1, dtype="c128", dist=UNIFORM, seed=0),
    "cfg2": dict(n=1 << 16, batch=1024, dtype="c128", dist=UNIFORM, seed=1),
    "cfg3": dict(n=1 << 28, batch=1, dtype="c128", dist=NORMAL, seed=2),
    "cfg4": dict(n=1 << 30, batch=1, dtype="c64", dist=UNIFORM, seed=3),
    "cfg5": dict(shape=(1024, 1024, 1024), dtype="c128", dist=NORMAL, seed=4),
}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.synth_draw.restype = ctypes.c_uint64
        lib.synth_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        for name in ("synth_fill_c128", "synth_fill_c64"):
            f = getattr(lib, name)
            f.restype = None
            f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int]
        _lib = lib
    return _lib


def draw(seed: int, c: int) -> int:
    return int(_load().synth_draw(seed, c))


def fill(count: int, seed: int, dist: int = UNIFORM, dtype: str = "c128", e0: int = 0,
         out: np.ndarray | None = None) -> np.ndarray:
    """Elements e0 .. e0+count-1 of the seeded stream as complex128/complex64."""
    npdt = np.complex128 if dtype == "c128" else np.complex64
    if out is None:
        out = np.empty(count, dtype=npdt)
    assert out.dtype == npdt and out.size == count and out.flags["C_CONTIGUOUS"]
    f = _load().synth_fill_c128 if dtype == "c128" else _load().synth_fill_c64
    f(out.ctypes.data, e0, count, seed, dist)
    return out


def config_input(name: str, e0: int = 0, count: int | None = None) -> np.ndarray:
    """A contiguous slice of the named config's input (global row-major index)."""
    c = CONFIGS[name]
    total = (c["shape"][0] * c["shape"][1] * c["shape"][2]) if "shape" in c else c["n"] * c["batch"]
    if count is None:
        count = total - e0
    return fill(count, c["seed"], c["dist"], c["dtype"], e0)

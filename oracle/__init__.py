"""oracle -- TEST INFRASTRUCTURE ONLY.

The CPU oracle of the hot path (PAPER.md, Mullin & Raynolds "Conformal
Computing"): oracle.c (the FFTs, the DFT definition and the Ch.3 lifted FFT,
complex128) and moa.py (the MoA/psi index algebra and every integer map).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  It shares no code with the CUDA path
(paper_0803_2386_b200/) and never imports it.

Pins: tests/test_oracle_*.py check every function here against what the paper
and the mathematics fix (printed worked examples under tests/golden/, closed
forms, invariants, brute force, numpy.fft as a third-party library routine).
Parity unpinned: none of the functions below.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

P64 = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, g++/gcc -O2 -fopenmp, no fast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        sig = {
            "orc_max_threads": [],
            "orc_bitrev_perm": [i64, vp],
            "orc_bitrev": [vp, i64],
            "orc_fft_radix2": [vp, i64],
            "orc_fft_radix2_batch": [vp, i64, i64],
            "orc_fft_radix2_sign": [vp, i64, ctypes.c_int],
            "orc_fft_radix2_batch_sign": [vp, i64, i64, ctypes.c_int],
            "orc_dft_direct": [vp, vp, i64],
            "orc_dft_direct_sign": [vp, vp, i64, ctypes.c_int],
            "orc_dft_bins": [vp, vp, i64, vp, vp, i64, vp],
            "orc_dft3_bins": [vp, i64, i64, i64, vp, i64, vp],
            "orc_reshape_transpose": [vp, vp, i64, i64],
            "orc_final_transpose": [vp, vp, i64, ctypes.c_int],
            "orc_lifted_plan": [i64, i64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
            "orc_fft_lifted": [vp, i64, i64],
            "orc_fft3d": [vp, i64, i64, i64],
            "orc_fft3d_sign": [vp, i64, i64, i64, ctypes.c_int],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = args
        _lib = lib
    return _lib


def _c128(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x), dtype=np.complex128)
    return a.copy() if a is x else a


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed (rc={rc})")


def max_threads() -> int:
    return int(_load().orc_max_threads())


def bitrev_perm(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    _check(_load().orc_bitrev_perm(n, out.ctypes.data), "bitrev_perm")
    return out


def bitrev(x) -> np.ndarray:
    a = _c128(x).copy()
    _check(_load().orc_bitrev(a.ctypes.data, a.size), "bitrev")
    return a


def fft_radix2(x) -> np.ndarray:
    """O1+O2: P_n then fftpsirad2 (forward sign); complex128 result."""
    a = _c128(x).copy()
    _check(_load().orc_fft_radix2(a.ctypes.data, a.size), "fft_radix2")
    return a


def fft_radix2_sign(x, sign: int) -> np.ndarray:
    """O1+O2 with kernel e^{sign 2 pi i jk/n}: sign=-1 forward; sign=+1 the
    fragment's EXP(+2 pi i row/L), the unnormalised inverse."""
    a = _c128(x).copy()
    _check(_load().orc_fft_radix2_sign(a.ctypes.data, a.size, sign), "fft_radix2_sign")
    return a


def fft_radix2_rows_sign(x, n: int, sign: int) -> np.ndarray:
    a = _c128(x).copy()
    assert a.size % n == 0
    _check(_load().orc_fft_radix2_batch_sign(a.ctypes.data, n, a.size // n, sign), "fft_radix2_batch_sign")
    return a


def dft_direct_sign(x, sign: int) -> np.ndarray:
    """O3 with kernel e^{sign 2 pi i jk/n}."""
    a = _c128(x)
    out = np.empty_like(a)
    _check(_load().orc_dft_direct_sign(a.ctypes.data, out.ctypes.data, a.size, sign), "dft_direct_sign")
    return out


def fft_radix2_inplace(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags["C_CONTIGUOUS"]
    _check(_load().orc_fft_radix2(a.ctypes.data, a.size), "fft_radix2")
    return a


def fft_radix2_rows(x, n: int) -> np.ndarray:
    a = _c128(x).copy()
    assert a.size % n == 0
    _check(_load().orc_fft_radix2_batch(a.ctypes.data, n, a.size // n), "fft_radix2_batch")
    return a


def fft_radix2_rows_inplace(a: np.ndarray, n: int) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags["C_CONTIGUOUS"] and a.size % n == 0
    _check(_load().orc_fft_radix2_batch(a.ctypes.data, n, a.size // n), "fft_radix2_batch")
    return a


def dft_direct(x) -> np.ndarray:
    """O3: the O(n^2) definition with exact integer exponent reduction."""
    a = _c128(x)
    out = np.empty_like(a)
    _check(_load().orc_dft_direct(a.ctypes.data, out.ctypes.data, a.size), "dft_direct")
    return out


def dft_bins(x: np.ndarray, n: int, bins, rows=None) -> np.ndarray:
    """O3 at selected bins: X[rows[i]][bins[i]] of the length-n rows of x
    (x complex128 or complex64; complex64 is promoted exactly)."""
    bins = np.ascontiguousarray(bins, dtype=np.int64)
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(bins.size, dtype=np.complex128)
    assert x.flags["C_CONTIGUOUS"]
    if x.dtype == np.complex64:
        px, p32 = None, x.ctypes.data
    else:
        assert x.dtype == np.complex128
        px, p32 = x.ctypes.data, None
    _check(_load().orc_dft_bins(px, p32, n, None if rows_a is None else rows_a.ctypes.data,
                                bins.ctypes.data, bins.size, out.ctypes.data), "dft_bins")
    return out


def dft3_bins(x: np.ndarray, shape, bins) -> np.ndarray:
    bins = np.ascontiguousarray(bins, dtype=np.int64).reshape(-1, 3)
    assert x.dtype == np.complex128 and x.flags["C_CONTIGUOUS"]
    out = np.empty(bins.shape[0], dtype=np.complex128)
    _check(_load().orc_dft3_bins(x.ctypes.data, shape[0], shape[1], shape[2], bins.ctypes.data,
                                 bins.shape[0], out.ctypes.data), "dft3_bins")
    return out


def reshape_transpose(x, c: int) -> np.ndarray:
    a = _c128(x)
    out = np.empty_like(a)
    _check(_load().orc_reshape_transpose(a.ctypes.data, out.ctypes.data, a.size, c), "reshape_transpose")
    return out


def final_transpose(x, sigma: int) -> np.ndarray:
    a = _c128(x)
    out = np.empty_like(a)
    _check(_load().orc_final_transpose(a.ctypes.data, out.ctypes.data, a.size, sigma), "final_transpose")
    return out


def lifted_plan(n: int, c: int):
    lm, pm = ctypes.c_int(), ctypes.c_int()
    _check(_load().orc_lifted_plan(n, c, ctypes.byref(lm), ctypes.byref(pm)), "lifted_plan")
    return lm.value, pm.value


def fft_lifted(x, c: int) -> np.ndarray:
    """O4: the paper's cache-optimized FFT with blocking size c."""
    a = _c128(x).copy()
    _check(_load().orc_fft_lifted(a.ctypes.data, a.size, c), "fft_lifted")
    return a


def fft3d(x) -> np.ndarray:
    """O5: row-major 3-D FFT by 1-D radix-2 FFTs along axes 2, 1, 0."""
    a = np.ascontiguousarray(np.asarray(x), dtype=np.complex128).copy()
    assert a.ndim == 3
    _check(_load().orc_fft3d(a.ctypes.data, *a.shape), "fft3d")
    return a


def fft3d_sign(x, sign: int) -> np.ndarray:
    """O5 with kernel e^{sign 2 pi i (...)} (sign=+1: the unnormalised inverse)."""
    a = np.ascontiguousarray(np.asarray(x), dtype=np.complex128).copy()
    assert a.ndim == 3
    _check(_load().orc_fft3d_sign(a.ctypes.data, *a.shape, sign), "fft3d_sign")
    return a


def fft3d_inplace(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.complex128 and a.ndim == 3 and a.flags["C_CONTIGUOUS"]
    _check(_load().orc_fft3d(a.ctypes.data, *a.shape), "fft3d")
    return a

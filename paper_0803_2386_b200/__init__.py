"""paper_0803_2386_b200 -- Python binding of libmoafft.so (include/moa_fft.h).

Argument marshalling only: every step of the FFT runs in the CUDA kernels of
csrc/.  The names follow the C-ABI.  PyTorch is used by callers for device
memory and streams; nothing here computes.  There is no CPU fallback: if the
extension is missing, importing this package raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmoafft.so")
# A/B measurements only: MOA_FFT_LIB_AB names another in-tree build of the
# same library (e.g. paper_0803_2386_b200/build/ab/libmoafft_prev.so)
if os.environ.get("MOA_FFT_LIB_AB"):
    _SO = os.path.join(os.path.dirname(_HERE), os.environ["MOA_FFT_LIB_AB"])

MOA_OK, MOA_EINVAL, MOA_ENOMEM, MOA_ECUDA, MOA_ENCCL, MOA_EUNSUPPORTED = range(6)
MOA_C64, MOA_C128 = 0, 1
MOA_FFT_INVERSE, MOA_FFT_NORMALIZE, MOA_FFT_LIFTED_ORDER, MOA_FFT_UNBLOCKED, MOA_FFT_HYPERCUBE = 1, 2, 4, 8, 16
MAX_DIGITS = 6
MAX_PASSES = 36
STATUS_NAMES = {0: "MOA_OK", 1: "MOA_EINVAL", 2: "MOA_ENOMEM", 3: "MOA_ECUDA", 4: "MOA_ENCCL",
                5: "MOA_EUNSUPPORTED"}

# every symbol include/moa_fft.h declares
EXPORTS = [
    "moa_fft_plan", "moa_fft_plan_lift", "moa_fft_plan_3d", "moa_fft_exec", "moa_fft_exec_host",
    "moa_fft_destroy", "moa_fft_last_error", "moa_fft_local_elems", "moa_fft_launches_per_exec",
    "moa_fft_get_unique_id", "moa_fft_dist_init", "moa_fft_dist_finalize", "moa_fft_dist_loopback",
    "moa_fft_exec_loopback", "moa_dist_describe", "moa_psi_describe", "moa_psi_describe_3d",
    "moa_plan_radices", "moa_fft_plan_describe", "moa_fft_prof_begin", "moa_fft_prof_end",
    "moa_fft_plan_ex", "moa_fft_plan_3d_ex", "moa_fft_output_index", "moa_pass_move",
    "moa_qgate_permutation", "moa_qgate_view_offset", "moa_qgate_apply",
]


class PassDesc(ctypes.Structure):
    """moa_pass_desc_t: one pass's ONF (see include/moa_fft.h)."""
    _fields_ = [
        ("logR", ctypes.c_int32), ("ndig", ctypes.c_int32),
        ("ext", ctypes.c_int64 * MAX_DIGITS), ("in_str", ctypes.c_int64 * MAX_DIGITS),
        ("out_str", ctypes.c_int64 * MAX_DIGITS), ("tw_str", ctypes.c_int64 * MAX_DIGITS),
        ("in_kstr", ctypes.c_int64), ("out_kstr", ctypes.c_int64),
        ("twN", ctypes.c_int64), ("tw_off", ctypes.c_int64),
        ("out_ksplit", ctypes.c_int32), ("out_kstr_hi", ctypes.c_int64),
        ("kind", ctypes.c_int32),
        ("lf_load", ctypes.c_int32), ("lf_store", ctypes.c_int32),
        ("W", ctypes.c_int32), ("threads", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
        ("line_pad", ctypes.c_int32), ("src", ctypes.c_int32), ("dst", ctypes.c_int32),
        ("ring", ctypes.c_int32), ("ring_slots", ctypes.c_int32), ("ring_lag", ctypes.c_int32),
        ("ring_discard", ctypes.c_int32), ("ring_groups", ctypes.c_int64), ("ring_G", ctypes.c_int64),
    ]

    @classmethod
    def from_dict(cls, d: dict) -> "PassDesc":
        s = cls()
        for name, _ in cls._fields_:
            if name in ("ext", "in_str", "out_str", "tw_str"):
                arr = getattr(s, name)
                for i, v in enumerate(d[name]):
                    arr[i] = v
            elif name in d:
                setattr(s, name, d[name])
        return s

    def to_dict(self) -> dict:
        nd = self.ndig
        return dict(logR=self.logR, R=1 << self.logR, ndig=nd, ext=list(self.ext[:nd]),
                    in_str=list(self.in_str[:nd]), out_str=list(self.out_str[:nd]),
                    tw_str=list(self.tw_str[:nd]), in_kstr=self.in_kstr, out_kstr=self.out_kstr,
                    twN=self.twN, tw_off=self.tw_off, out_ksplit=self.out_ksplit,
                    out_kstr_hi=self.out_kstr_hi, kind=self.kind, lf_load=self.lf_load,
                    lf_store=self.lf_store, W=self.W, threads=self.threads,
                    smem_bytes=self.smem_bytes, line_pad=self.line_pad, src=self.src, dst=self.dst,
                    ring=self.ring, ring_slots=self.ring_slots, ring_lag=self.ring_lag,
                    ring_discard=self.ring_discard, ring_groups=self.ring_groups, ring_G=self.ring_G)


class MoaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: build it with __graft_entry__.build() "
                          "(python -m paper_0803_2386_b200._build); there is no CPU fallback")
    lib = ctypes.CDLL(_SO)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P = ctypes.POINTER
    sig = {
        "moa_fft_plan": [P(vp), i64, i64, i32, i32],
        "moa_fft_plan_lift": [P(vp), i64, i64, i32, P(i64), i32],
        "moa_fft_plan_3d": [P(vp), i64, i64, i64, i32, i32],
        "moa_fft_plan_ex": [P(vp), i64, i64, i32, i32, ctypes.c_uint32],
        "moa_fft_plan_3d_ex": [P(vp), i64, i64, i64, i32, i32, ctypes.c_uint32],
        "moa_fft_output_index": [vp, P(i64), i64],
        "moa_pass_move": [P(PassDesc), i32, vp, vp, vp],
        "moa_qgate_permutation": [i32, P(ctypes.c_int32), i32, P(ctypes.c_int32)],
        "moa_qgate_view_offset": [i32, P(ctypes.c_int32), i32, i64, i64, P(i64)],
        "moa_qgate_apply": [vp, i32, P(ctypes.c_int32), i32, vp, i32, vp],
        "moa_fft_exec": [vp, vp, vp, vp],
        "moa_fft_exec_host": [vp, vp, vp, vp],
        "moa_fft_destroy": [vp],
        "moa_fft_get_unique_id": [P(ctypes.c_uint8)],
        "moa_fft_dist_init": [i32, i32, P(ctypes.c_uint8)],
        "moa_fft_dist_finalize": [],
        "moa_fft_dist_loopback": [i32, i32],
        "moa_fft_exec_loopback": [P(vp), i32, P(vp), P(vp), vp],
        "moa_dist_describe": [i32, i32, i32, i64, i64, i64, i32, vp, i32, P(i32), P(ctypes.c_int32),
                              P(ctypes.c_int32), P(ctypes.c_int32), P(i64), i32, P(i32), ctypes.c_uint32],
        "moa_psi_describe": [i64, i64, i32, P(i64), i32, P(PassDesc), i32, P(i32)],
        "moa_psi_describe_3d": [i64, i64, i64, i32, P(PassDesc), i32, P(i32)],
        "moa_plan_radices": [i64, i64, i32, P(i64), i32, P(i32)],
        "moa_fft_plan_describe": [vp, P(PassDesc), i32, P(i32)],
        "moa_fft_prof_begin": [vp, i32],
        "moa_fft_prof_end": [vp, P(ctypes.c_double), i32, P(i32), P(i32)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.moa_fft_last_error.argtypes = []
    lib.moa_fft_last_error.restype = ctypes.c_char_p
    lib.moa_fft_local_elems.argtypes = [vp]
    lib.moa_fft_local_elems.restype = i64
    lib.moa_fft_launches_per_exec.argtypes = [vp]
    lib.moa_fft_launches_per_exec.restype = ctypes.c_int
    return lib


lib = _load()


def _check(st: int):
    if st != MOA_OK:
        raise MoaError(st, lib.moa_fft_last_error().decode())


def _dt(dtype) -> int:
    if dtype in (MOA_C64, "c64", "complex64"):
        return MOA_C64
    if dtype in (MOA_C128, "c128", "complex128"):
        return MOA_C128
    if hasattr(dtype, "is_complex"):  # torch dtype
        import torch
        return MOA_C64 if dtype == torch.complex64 else MOA_C128
    raise ValueError(f"unknown dtype {dtype!r}")


# ---------------------------------------------------------------- C-ABI names
def moa_fft_plan(n: int, batch: int = 1, dtype="c128", ngpu: int = 1) -> int:
    h = ctypes.c_void_p()
    _check(lib.moa_fft_plan(ctypes.byref(h), n, batch, _dt(dtype), ngpu))
    return h.value


def moa_fft_plan_ex(n: int, batch: int = 1, dtype="c128", ngpu: int = 1, flags: int = 0) -> int:
    h = ctypes.c_void_p()
    _check(lib.moa_fft_plan_ex(ctypes.byref(h), n, batch, _dt(dtype), ngpu, flags))
    return h.value


def moa_fft_plan_3d_ex(n0: int, n1: int, n2: int, dtype="c128", ngpu: int = 1, flags: int = 0) -> int:
    h = ctypes.c_void_p()
    _check(lib.moa_fft_plan_3d_ex(ctypes.byref(h), n0, n1, n2, _dt(dtype), ngpu, flags))
    return h.value


def moa_fft_output_index(plan: int, n: int):
    """pos[k] = offset where X[k] is stored (see include/moa_fft.h)."""
    import numpy as np
    pos = np.empty(n, dtype=np.int64)
    _check(lib.moa_fft_output_index(plan, pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n))
    return pos


def moa_pass_move(desc: dict, dtype, in_ptr: int, out_ptr: int, stream: int = 0) -> None:
    """Test hook: run one pass descriptor (a dict from moa_psi_describe*) as a
    pure data movement on the GPU (see include/moa_fft.h)."""
    d = PassDesc.from_dict(desc)
    _check(lib.moa_pass_move(ctypes.byref(d), _dt(dtype), in_ptr, out_ptr, stream))


def moa_qgate_permutation(n: int, gated_bits) -> list:
    """The Ch.6 transpose vector t (2n entries) moving the gated bits to the diagonal."""
    bits = (ctypes.c_int32 * len(gated_bits))(*gated_bits)
    t = (ctypes.c_int32 * (2 * n))()
    _check(lib.moa_qgate_permutation(n, bits, len(gated_bits), t))
    return list(t)


def moa_qgate_view_offset(n: int, gated_bits, view_row: int, view_col: int) -> int:
    bits = (ctypes.c_int32 * len(gated_bits))(*gated_bits)
    off = ctypes.c_int64()
    _check(lib.moa_qgate_view_offset(n, bits, len(gated_bits), view_row, view_col, ctypes.byref(off)))
    return off.value


def moa_qgate_apply(rho, n: int, gated_bits, u, stream=None) -> None:
    """D <- U_full D U_full^dagger in place on the CUDA tensor rho (2^n x 2^n,
    complex64/complex128); u: the 2^q x 2^q gate (numpy / host)."""
    import numpy as np
    import torch
    if rho.dtype not in (torch.complex64, torch.complex128) or not rho.is_cuda or not rho.is_contiguous():
        raise ValueError("qgate: rho must be a contiguous CUDA complex64 / complex128 tensor")
    if tuple(rho.shape) != (1 << n, 1 << n):
        raise ValueError(f"qgate: rho must be 2^n x 2^n = {(1 << n, 1 << n)}, got {tuple(rho.shape)}")
    dt = MOA_C128 if rho.dtype == torch.complex128 else MOA_C64
    uh = np.ascontiguousarray(u, dtype=np.complex128 if dt == MOA_C128 else np.complex64)
    q = len(gated_bits)
    if uh.shape != (1 << q, 1 << q):
        raise ValueError(f"qgate: u must be 2^q x 2^q = {(1 << q, 1 << q)} for {q} gated bits, got {uh.shape}")
    bits = (ctypes.c_int32 * len(gated_bits))(*gated_bits)
    s = stream if stream is not None else torch.cuda.current_stream(rho.device)
    _check(lib.moa_qgate_apply(rho.data_ptr(), n, bits, len(gated_bits), uh.ctypes.data, dt, s.cuda_stream))


def moa_fft_plan_lift(n: int, batch: int, dtype, radices) -> int:
    h = ctypes.c_void_p()
    arr = (ctypes.c_int64 * len(radices))(*radices)
    _check(lib.moa_fft_plan_lift(ctypes.byref(h), n, batch, _dt(dtype), arr, len(radices)))
    return h.value


def moa_fft_plan_3d(n0: int, n1: int, n2: int, dtype="c128", ngpu: int = 1) -> int:
    h = ctypes.c_void_p()
    _check(lib.moa_fft_plan_3d(ctypes.byref(h), n0, n1, n2, _dt(dtype), ngpu))
    return h.value


def moa_fft_exec(plan: int, in_ptr: int, out_ptr: int, stream: int = 0) -> None:
    _check(lib.moa_fft_exec(plan, in_ptr, out_ptr, stream))


def moa_fft_exec_host(plan: int, in_ptr: int, out_ptr: int, stream: int = 0) -> None:
    _check(lib.moa_fft_exec_host(plan, in_ptr, out_ptr, stream))


def moa_fft_destroy(plan: int) -> None:
    _check(lib.moa_fft_destroy(plan))


def moa_fft_last_error() -> str:
    return lib.moa_fft_last_error().decode()


def moa_fft_local_elems(plan: int) -> int:
    return int(lib.moa_fft_local_elems(plan))


def moa_fft_launches_per_exec(plan: int) -> int:
    return int(lib.moa_fft_launches_per_exec(plan))


def _default_nccl_lib() -> None:
    # Point the C side at the NCCL wheel next to torch (2.28: has ncclAlltoAll)
    # unless the caller chose one; without it the C side falls back to the
    # search path and, on an older NCCL, to grouped ncclSend / ncclRecv.
    if os.environ.get("MOA_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for d in (spec.submodule_search_locations if spec else []):
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["MOA_NCCL_LIB"] = cand
            return


def moa_fft_get_unique_id() -> bytes:
    _default_nccl_lib()
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.moa_fft_get_unique_id(buf))
    return bytes(buf)


def moa_fft_dist_init(rank: int, ngpu: int, uid: bytes) -> None:
    _default_nccl_lib()
    buf = (ctypes.c_uint8 * 128)(*uid)
    _check(lib.moa_fft_dist_init(rank, ngpu, buf))


def moa_fft_dist_finalize() -> None:
    _check(lib.moa_fft_dist_finalize())


def moa_fft_dist_loopback(rank: int, ngpu: int) -> None:
    _check(lib.moa_fft_dist_loopback(rank, ngpu))


def moa_fft_exec_loopback(plans, ins, outs, stream: int = 0) -> None:
    p = len(plans)
    _check(lib.moa_fft_exec_loopback((ctypes.c_void_p * p)(*plans), p, (ctypes.c_void_p * p)(*ins),
                                     (ctypes.c_void_p * p)(*outs), stream))


def moa_psi_describe(n: int, batch: int = 1, dtype="c128", radices=None) -> list:
    out = (PassDesc * MAX_PASSES)()
    np_ = ctypes.c_int()
    arr = (ctypes.c_int64 * len(radices))(*radices) if radices else None
    _check(lib.moa_psi_describe(n, batch, _dt(dtype), arr, len(radices) if radices else 0, out, MAX_PASSES,
                                ctypes.byref(np_)))
    return [out[i].to_dict() for i in range(np_.value)]


def moa_psi_describe_3d(n0: int, n1: int, n2: int, dtype="c128") -> list:
    out = (PassDesc * MAX_PASSES)()
    np_ = ctypes.c_int()
    _check(lib.moa_psi_describe_3d(n0, n1, n2, _dt(dtype), out, MAX_PASSES, ctypes.byref(np_)))
    return [out[i].to_dict() for i in range(np_.value)]


def moa_plan_radices(n: int, batch: int = 1, dtype="c128") -> list:
    arr = (ctypes.c_int64 * 32)()
    nr = ctypes.c_int()
    _check(lib.moa_plan_radices(n, batch, _dt(dtype), arr, 32, ctypes.byref(nr)))
    return list(arr[: nr.value])


def moa_fft_plan_describe(plan: int) -> list:
    out = (PassDesc * MAX_PASSES)()
    np_ = ctypes.c_int()
    _check(lib.moa_fft_plan_describe(plan, out, MAX_PASSES, ctypes.byref(np_)))
    return [out[i].to_dict() for i in range(np_.value)]


def moa_fft_prof_begin(plan: int, max_execs: int) -> None:
    _check(lib.moa_fft_prof_begin(plan, max_execs))


def moa_fft_prof_end(plan: int):
    """-> (summed ms per step over the recorded execs, number of execs)."""
    arr = (ctypes.c_double * 64)()
    ns, nx = ctypes.c_int(), ctypes.c_int()
    _check(lib.moa_fft_prof_end(plan, arr, 64, ctypes.byref(ns), ctypes.byref(nx)))
    return list(arr[: ns.value]), nx.value


def moa_dist_describe(rank: int, ngpu: int, n, dtype="c128", flags: int = 0) -> dict:
    """Schedule of one rank: n = N (1-D) or (n0, n1, n2) (3-D slab)."""
    is3d = isinstance(n, (tuple, list))
    n0, n1, n2 = (n if is3d else (n, 0, 0))
    passes = (PassDesc * MAX_PASSES)()
    np_, ns = ctypes.c_int(), ctypes.c_int()
    kinds, srcs, dsts = (ctypes.c_int32 * 32)(), (ctypes.c_int32 * 32)(), (ctypes.c_int32 * 32)()
    counts = (ctypes.c_int64 * 32)()
    _check(lib.moa_dist_describe(rank, ngpu, int(is3d), n0, n1, n2, _dt(dtype), ctypes.cast(passes, ctypes.c_void_p),
                                 MAX_PASSES, ctypes.byref(np_), kinds, srcs, dsts, counts, 32, ctypes.byref(ns),
                                 flags))
    steps = []
    for i in range(ns.value):
        if kinds[i] == 0:
            steps.append(("pass", srcs[i]))
        elif kinds[i] == 1:
            steps.append(("alltoall", srcs[i], dsts[i], counts[i]))
        elif kinds[i] == 2:
            steps.append(("fused", srcs[i], dsts[i], counts[i]))      # pass + all-to-all by its stores
        else:
            steps.append(("barrier",))
    return dict(passes=[passes[i].to_dict() for i in range(np_.value)], steps=steps)


# ---------------------------------------------------------------- convenience
class FFTPlan:
    """RAII wrapper: FFTPlan(n, batch, dtype) or FFTPlan.plan_3d(...); exec on
    torch device tensors (complex64 / complex128, contiguous)."""

    def __init__(self, n: int = 0, batch: int = 1, dtype="c128", ngpu: int = 1, radices=None, _handle=None,
                 inverse: bool = False, normalize: bool = False, lifted_order: bool = False,
                 unblocked: bool = False, hypercube: bool = False):
        flags = (MOA_FFT_INVERSE if inverse else 0) | (MOA_FFT_NORMALIZE if normalize else 0) | \
            (MOA_FFT_LIFTED_ORDER if lifted_order else 0) | (MOA_FFT_UNBLOCKED if unblocked else 0) | \
            (MOA_FFT_HYPERCUBE if hypercube else 0)
        if _handle is not None:
            self.h = _handle
        elif radices is not None:
            if flags:
                raise ValueError("explicit radices take no flags")
            self.h = moa_fft_plan_lift(n, batch, dtype, radices)
        else:
            self.h = moa_fft_plan_ex(n, batch, dtype, ngpu, flags)
        self.dtype = _dt(dtype)
        self.n = n

    @classmethod
    def plan_3d(cls, n0, n1, n2, dtype="c128", ngpu: int = 1, inverse: bool = False, normalize: bool = False):
        flags = (MOA_FFT_INVERSE if inverse else 0) | (MOA_FFT_NORMALIZE if normalize else 0)
        return cls(_handle=moa_fft_plan_3d_ex(n0, n1, n2, dtype, ngpu, flags), dtype=dtype)

    def output_index(self):
        """pos[k]: where X[k] is stored (identity for natural order)."""
        return moa_fft_output_index(self.h, self.n)

    @property
    def local_elems(self) -> int:
        return moa_fft_local_elems(self.h)

    @property
    def launches(self) -> int:
        return moa_fft_launches_per_exec(self.h)

    def describe(self) -> list:
        return moa_fft_plan_describe(self.h)

    def exec(self, x, out=None, stream=None):
        import torch
        want = torch.complex64 if self.dtype == MOA_C64 else torch.complex128
        if x.dtype != want or not x.is_cuda or not x.is_contiguous():
            raise ValueError(f"exec: expected a contiguous CUDA {want} tensor")
        if x.numel() != self.local_elems:
            raise ValueError(f"exec: expected {self.local_elems} elements, got {x.numel()}")
        if out is None:
            out = torch.empty_like(x)
        elif (out.dtype != want or out.device != x.device or not out.is_contiguous()
              or out.numel() != self.local_elems):
            raise ValueError(f"exec: out must be a contiguous {want} tensor of {self.local_elems} elements "
                             f"on {x.device}")
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        moa_fft_exec(self.h, x.data_ptr(), out.data_ptr(), s.cuda_stream)
        return out

    def exec_host(self, x_host, out_host, stream=None):
        """End-to-end: host (pinned) buffers in and out; synchronises."""
        import torch
        want = torch.complex64 if self.dtype == MOA_C64 else torch.complex128
        for name, t in (("x_host", x_host), ("out_host", out_host)):
            if t.is_cuda or t.dtype != want or not t.is_contiguous() or t.numel() != self.local_elems:
                raise ValueError(f"exec_host: {name} must be a contiguous host {want} tensor of "
                                 f"{self.local_elems} elements")
        s = stream if stream is not None else torch.cuda.current_stream()
        moa_fft_exec_host(self.h, x_host.data_ptr(), out_host.data_ptr(), s.cuda_stream)
        return out_host

    def close(self):
        if getattr(self, "h", None):
            moa_fft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

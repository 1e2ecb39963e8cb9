"""paper_2103_02605_b200 — thin Python binding of libfcirc (include/fcirc.h).

Argument marshalling only: every step of the f-circulant product (arXiv 2103.02605, Theorem 1 /
Algorithm 1) runs in the sm_100a kernels of ``lib/libfcirc.so``.  PyTorch is used for
device memory and streams.  There is no CPU fallback: if the library is missing this module raises.

Functions mirror the C ABI names:
  matvec(a, b, f, p, out=None)      -> fcirc_matvec       (device tensors [batch, n])
  matvec_host(a, b, f, p, out=None) -> fcirc_matvec_host  (host arrays/tensors, pinned preferred)
  circulant_matvec(a, b, p)         -> fcirc_circulant_matvec (f = 1, any order n: Corollary 1)
  polymul(a, b, p, out=None)        -> fcirc_polymul      (device tensors [batch, na], [batch, nb])
  bigint_mul(x, y, out=None)        -> bigint_mul         (device uint32 words [batch, nx], [batch, ny])
  plan_table(p, f, n)               -> fcirc_plan_table   (host-only twist-table inspection)
  primitive_rate(kind)              -> fcirc_primitive_rate (measured rate of the ring primitives)
  plan_count()                      -> fcirc_plan_count   (cached / graph-pinned plans)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["FcircError", "matvec", "matvec_host", "circulant_matvec", "polymul", "bigint_mul", "plan_table", "strerror",
           "last_launch_count", "release_cache", "plan_count", "primitive_rate", "version", "library_path", "schedule", "P998", "P469", "P167",
           "GOLDILOCKS", "PRIMES", "M31X2", "fp2_pack"]

P998 = 998244353
P469 = 469762049
P167 = 167772161
GOLDILOCKS = (1 << 64) - (1 << 32) + 1
PRIMES = (P998, P469, P167, GOLDILOCKS)
# The paper's own ring Z/pZ[sqrt 3], p = 2^31 - 1: pass p = M31X2; elements u + v sqrt 3 are
# uint64 packed u | v << 32 (fp2_pack), including the scalar f.
M31X2 = (1 << 31) - 1


def fp2_pack(u: int, v: int) -> int:
    """u + v sqrt 3 in Z/(2^31 - 1)[sqrt 3] -> the packed 64-bit element (u, v canonical)."""
    return (int(u) % M31X2) | ((int(v) % M31X2) << 32)

_HERE = os.path.dirname(os.path.abspath(__file__))
# FCIRC_LIB: an alternative build of the same library (A/B experiments, tools/gpu_sweep.sh)
_LIB_PATH = os.environ.get("FCIRC_LIB") or os.path.join(_HERE, "lib", "libfcirc.so")
_lib = None


def library_path() -> str:
    return _LIB_PATH


class FcircError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} (status {code})")


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"libfcirc.so not built at {_LIB_PATH}; run `python __graft_entry__.py build` "
                           "(no CPU fallback exists)")
    lib = ctypes.CDLL(_LIB_PATH)
    u64, i64, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
    lib.fcirc_matvec.argtypes = [u64, u64, vp, vp, vp, i64, i64, vp]
    lib.fcirc_matvec_host.argtypes = [u64, u64, vp, vp, vp, i64, i64]
    lib.fcirc_circulant_matvec.argtypes = [u64, vp, vp, vp, i64, i64, vp]
    lib.fcirc_polymul.argtypes = [u64, vp, i64, vp, i64, vp, i64, vp]
    lib.bigint_mul.argtypes = [vp, i64, vp, i64, vp, i64, vp]
    lib.fcirc_plan_table.argtypes = [u64, u64, i64, vp, vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    lib.fcirc_schedule.argtypes = [u64, i64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    lib.fcirc_profile_enable.argtypes = [ctypes.c_int]
    lib.fcirc_profile_read.argtypes = [vp, vp, ctypes.c_int]
    lib.fcirc_primitive_rate.argtypes = [ctypes.c_int, i64, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double), vp]
    lib.fcirc_primitive_rate.restype = ctypes.c_int
    lib.fcirc_plan_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.fcirc_plan_count.restype = i64
    for fn in (lib.fcirc_matvec, lib.fcirc_matvec_host, lib.fcirc_circulant_matvec, lib.fcirc_polymul, lib.bigint_mul, lib.fcirc_plan_table,
               lib.fcirc_schedule,
               lib.fcirc_release_cache, lib.fcirc_profile_enable, lib.fcirc_profile_read):
        fn.restype = ctypes.c_int
    lib.fcirc_strerror.argtypes = [ctypes.c_int]
    lib.fcirc_strerror.restype = ctypes.c_char_p
    lib.fcirc_version.restype = ctypes.c_char_p
    lib.fcirc_last_launch_count.restype = i64
    _lib = lib
    return lib


def strerror(code: int) -> str:
    return _load().fcirc_strerror(int(code)).decode()


def version() -> str:
    return _load().fcirc_version().decode()


def last_launch_count() -> int:
    return int(_load().fcirc_last_launch_count())


KERNEL_KINDS = ("k_block_fused", "k_block_sub", "k_cols_fwd", "k_cols_inv", "apps")


def profile_enable(on: bool = True) -> None:
    """Bracket every libfcirc launch with CUDA events on its stream (fcirc_profile_enable)."""
    _load().fcirc_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kind: (launches, device ms)} accumulated since the last read (fcirc_profile_read)."""
    counts = np.zeros(len(KERNEL_KINDS), dtype=np.int64)
    ms = np.zeros(len(KERNEL_KINDS), dtype=np.float64)
    rc = _load().fcirc_profile_read(counts.ctypes.data, ms.ctypes.data, len(KERNEL_KINDS))
    if rc < 0:
        raise FcircError(rc, "fcirc_profile_read")
    return {k: (int(c), float(t)) for k, c, t in zip(KERNEL_KINDS, counts, ms)}


def release_cache() -> None:
    _load().fcirc_release_cache()


def plan_count():
    """(cached plans, of which pinned by CUDA-graph captures) -- fcirc_plan_count."""
    pinned = ctypes.c_int(0)
    n = _load().fcirc_plan_count(ctypes.byref(pinned))
    return int(n), int(pinned.value)


PRIMITIVES = {"gold_mul": 0, "gold_fwd_a": 1, "gold_fwd_b": 2, "gold_inv": 3, "u32_mulc": 4, "u32_leaf": 5,
              "u32_fwd_a": 6, "imad_wide": 7, "m31x2_mul": 8,
              "gold_mulm": 9, "gold_leaf": 10}


def primitive_rate(kind: str, iters: int = 20000, stream=None):
    """(primitives per second, ms of the timed launch) of one of the library's own ring primitives
    on all SMs of the current device (fcirc_primitive_rate; synchronises the stream)."""
    torch = _torch()
    ops = ctypes.c_double(0.0)
    ms = ctypes.c_double(0.0)
    dev = torch.device("cuda", torch.cuda.current_device())
    rc = _load().fcirc_primitive_rate(PRIMITIVES[kind], int(iters), ctypes.byref(ops), ctypes.byref(ms),
                                      _stream_handle(stream, dev))
    _check(rc, "fcirc_primitive_rate")
    return float(ops.value), float(ms.value)


def _check(rc: int, where: str):
    if rc != 0:
        raise FcircError(rc, where)


def _elem_bytes(p: int) -> int:
    return 8 if int(p) >= (1 << 32) or int(p) == M31X2 else 4


def _scalar(f: int, p: int) -> int:
    """f reduced mod p; packed Z/p[sqrt 3] scalars are passed as they are."""
    return int(f) if int(p) == M31X2 else int(f) % int(p)


def _torch():
    import torch
    return torch


def _dev_tensor(x, p: int, name: str):
    torch = _torch()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.element_size() != _elem_bytes(p) or x.dtype.is_floating_point:
        raise TypeError(f"{name}: element type must be a {8 * _elem_bytes(p)}-bit integer for p={p}")
    if not x.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return x


def _same_device(ref, *others):
    for name, x in others:
        if x.device != ref.device:
            raise ValueError(f"{name} is on {x.device}, expected {ref.device} (all operands on one GPU)")


def _check_out(out, shape, p: int, name: str = "out"):
    _dev_tensor(out, p, name)
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(out.shape)}, expected {tuple(shape)}")
    return out


def _stream_handle(stream, device):
    """The stream the library launches on: the given one (must belong to `device`) or `device`'s
    current stream."""
    torch = _torch()
    if stream is None:
        s = torch.cuda.current_stream(device)
    else:
        s = stream
        if s.device != device:
            raise ValueError(f"stream belongs to {s.device}, operands to {device}")
    return ctypes.c_void_p(s.cuda_stream)


def matvec(a, b, f: int, p: int, out=None, stream=None):
    """c = A b for f-circulant A with first row ``a`` (Definition 2), batched.

    ``a``, ``b``: CUDA tensors [batch, n] (or [n]) of uint32/int32 (32-bit primes) or uint64/int64
    (Goldilocks) holding canonical residues.  Returns ``out`` (allocated if None), same shape.
    Asynchronous on the current (or given) stream.
    """
    torch = _torch()
    _dev_tensor(a, p, "a")
    _dev_tensor(b, p, "b")
    if a.shape != b.shape:
        raise ValueError("a and b must have the same shape")
    n = a.shape[-1]
    batch = a.numel() // n if n else 0
    if out is None:
        out = torch.empty_like(a)
    _check_out(out, a.shape, p)
    _same_device(a, ("b", b), ("out", out))
    with torch.cuda.device(a.device):   # the library launches on the current device
        rc = _load().fcirc_matvec(int(p), _scalar(f, p), a.data_ptr(), b.data_ptr(), out.data_ptr(), n, batch,
                                  _stream_handle(stream, a.device))
    _check(rc, "fcirc_matvec")
    return out


def circulant_matvec(a, b, p: int, out=None, stream=None):
    """c = A b for usual circulants (f = 1) of ANY order n (Corollary 1), batched.

    ``a``, ``b``: CUDA tensors [batch, n] of residues (element type as in ``matvec``).
    """
    torch = _torch()
    _dev_tensor(a, p, "a")
    _dev_tensor(b, p, "b")
    if a.shape != b.shape:
        raise ValueError("a and b must have the same shape")
    n = a.shape[-1]
    batch = a.numel() // n if n else 0
    if out is None:
        out = torch.empty_like(a)
    _check_out(out, a.shape, p)
    _same_device(a, ("b", b), ("out", out))
    with torch.cuda.device(a.device):
        rc = _load().fcirc_circulant_matvec(int(p), a.data_ptr(), b.data_ptr(), out.data_ptr(), n, batch,
                                            _stream_handle(stream, a.device))
    _check(rc, "fcirc_circulant_matvec")
    return out


def _host_ptr(x, p: int, name: str):
    torch = _torch()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"] or x.itemsize != _elem_bytes(p):
            raise TypeError(f"{name}: contiguous {8 * _elem_bytes(p)}-bit integer array required")
        return x.ctypes.data, x.shape
    if isinstance(x, torch.Tensor) and not x.is_cuda:
        if not x.is_contiguous() or x.element_size() != _elem_bytes(p):
            raise TypeError(f"{name}: contiguous {8 * _elem_bytes(p)}-bit integer tensor required")
        return x.data_ptr(), tuple(x.shape)
    raise TypeError(f"{name} must be a host numpy array or CPU tensor")


def matvec_host(a, b, f: int, p: int, out=None):
    """fcirc_matvec_host: host buffers in, host buffer out (H2D, kernels, D2H pipelined)."""
    pa, sa = _host_ptr(a, p, "a")
    pb, sb = _host_ptr(b, p, "b")
    if tuple(sa) != tuple(sb):
        raise ValueError("a and b must have the same shape")
    if out is None:
        out = np.empty(sa, dtype=np.uint64 if _elem_bytes(p) == 8 else np.uint32)
    pc, sc = _host_ptr(out, p, "out")
    if tuple(sc) != tuple(sa):
        raise ValueError(f"out has shape {tuple(sc)}, expected {tuple(sa)}")
    n = sa[-1]
    batch = int(np.prod(sa)) // n
    rc = _load().fcirc_matvec_host(int(p), _scalar(f, p), pa, pb, pc, n, batch)
    _check(rc, "fcirc_matvec_host")
    return out


def polymul(a, b, p: int, out=None, stream=None):
    """c = a(x) b(x) mod p for device tensors [batch, na], [batch, nb] -> [batch, na+nb-1]."""
    torch = _torch()
    _dev_tensor(a, p, "a")
    _dev_tensor(b, p, "b")
    na, nb = a.shape[-1], b.shape[-1]
    batch = a.numel() // na
    if b.numel() // nb != batch:
        raise ValueError("a and b must have the same batch")
    if out is None:
        out = torch.empty((*a.shape[:-1], na + nb - 1), dtype=a.dtype, device=a.device)
    _check_out(out, (*a.shape[:-1], na + nb - 1), p)
    _same_device(a, ("b", b), ("out", out))
    with torch.cuda.device(a.device):
        rc = _load().fcirc_polymul(int(p), a.data_ptr(), na, b.data_ptr(), nb, out.data_ptr(), batch,
                                   _stream_handle(stream, a.device))
    _check(rc, "fcirc_polymul")
    return out


def bigint_mul(x, y, out=None, stream=None):
    """z = x * y for little-endian uint32 word tensors [batch, nx], [batch, ny] -> [batch, nx+ny]."""
    torch = _torch()
    _dev_tensor(x, P998, "x")
    _dev_tensor(y, P998, "y")
    nx, ny = x.shape[-1], y.shape[-1]
    batch = x.numel() // nx
    if y.numel() // ny != batch:
        raise ValueError("x and y must have the same batch")
    if out is None:
        out = torch.empty((*x.shape[:-1], nx + ny), dtype=x.dtype, device=x.device)
    _check_out(out, (*x.shape[:-1], nx + ny), P998)
    _same_device(x, ("y", y), ("out", out))
    with torch.cuda.device(x.device):
        rc = _load().bigint_mul(x.data_ptr(), nx, y.data_ptr(), ny, out.data_ptr(), batch,
                                _stream_handle(stream, x.device))
    _check(rc, "bigint_mul")
    return out


def schedule(p: int, n: int):
    """Host-only: (log2 of the on-chip sub-problem size, number of column-pass levels) that
    fcirc_matvec uses for (p, n) (fcirc_schedule)."""
    m = ctypes.c_int(0)
    k = ctypes.c_int(0)
    _check(_load().fcirc_schedule(int(p), int(n), ctypes.byref(m), ctypes.byref(k)), "fcirc_schedule")
    return int(m.value), int(k.value)


def plan_table(p: int, f: int, n: int):
    """Host-only: (s, sinv, w, K) of the twist table the library would use for (p, f, n)."""
    size = max(int(n), 1)
    s = np.zeros(size, dtype=np.uint64)
    si = np.zeros(size, dtype=np.uint64)
    w = ctypes.c_uint64(0)
    K = ctypes.c_uint64(0)
    rc = _load().fcirc_plan_table(int(p), _scalar(f, p), int(n), s.ctypes.data, si.ctypes.data,
                                  ctypes.byref(w), ctypes.byref(K))
    _check(rc, "fcirc_plan_table")
    return s, si, int(w.value), int(K.value)

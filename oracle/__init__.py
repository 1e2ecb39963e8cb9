"""oracle — the plain CPU oracle for libfcirc (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2103_02605_b200`` never imports it and shares no code with it.

Contents (each cites the PAPER.md line it follows, ``P:n``):

* ``fcirc_entries``  — c_i of the f-circulant product straight from Definition 2
   with the row-vector identification: the C library ``liboracle.so``
  (``oracle.c``), O(n) per entry, exact 192-bit accumulation.
* ``polymul_coeffs`` — schoolbook polynomial coefficients, C library.
* ``fcirc_entries_batch`` / ``poly_eval_batch`` — the same definitions over a whole
  ``[batch][n]`` array (per-instance index / point lists), threaded; indexing only.
* ``bigint_mul``     — independent Karatsuba on 32-bit words, C library.
* ``py_fcirc_matvec`` — second witness for ``fcirc_entries``: the same definition in
  arbitrary-precision Python ints (no ``%`` tricks), for small n.
* ``materialize``    — literal application of rules (1) and (2) of Definition 2
   starting from the first row; a different code path from the index formula.
* ``alg1_recursive`` — literal Algorithm 1 applied recursively with
  caller-chosen (e.g. random) square-root signs; used only as a pin that the method
  reaches the definition (Theorem 1), never as the oracle itself.

Every function is pinned by ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with plain gcc (no CUDA)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i64p = ctypes.POINTER(ctypes.c_int64)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_fcirc_entries.argtypes = [ctypes.c_uint64, ctypes.c_uint64, u64p, u64p, ctypes.c_int64,
                                             i64p, ctypes.c_int64, u64p, ctypes.c_int]
        lib.oracle_polymul_coeffs.argtypes = [ctypes.c_uint64, u64p, ctypes.c_int64, u64p, ctypes.c_int64,
                                              i64p, ctypes.c_int64, u64p, ctypes.c_int]
        lib.oracle_poly_eval.argtypes = [ctypes.c_uint64, u64p, ctypes.c_int64, u64p, ctypes.c_int64, u64p,
                                         ctypes.c_int]
        lib.oracle_poly_eval.restype = ctypes.c_int
        lib.oracle_bigint_mul.argtypes = [u32p, ctypes.c_int64, u32p, ctypes.c_int64, u32p]
        lib.oracle_fcirc_entries_m31x2.argtypes = [ctypes.c_uint64, u64p, u64p, ctypes.c_int64, i64p, ctypes.c_int64,
                                                   u64p, ctypes.c_int]
        lib.oracle_polymul_coeffs_m31x2.argtypes = [u64p, ctypes.c_int64, u64p, ctypes.c_int64, i64p, ctypes.c_int64,
                                                    u64p, ctypes.c_int]
        lib.oracle_bigint_mul_school.argtypes = [u32p, ctypes.c_int64, u32p, ctypes.c_int64, u32p]
        lib.oracle_fcirc_entries_batch.argtypes = [ctypes.c_uint64, ctypes.c_uint64, u64p, u64p, ctypes.c_int64,
                                                   ctypes.c_int64, i64p, ctypes.c_int64, u64p, ctypes.c_int]
        lib.oracle_poly_eval_batch.argtypes = [ctypes.c_uint64, u64p, ctypes.c_int64, ctypes.c_int64, u64p,
                                               ctypes.c_int64, u64p, ctypes.c_int]
        lib.oracle_fcirc_entries_batch.restype = ctypes.c_int
        lib.oracle_poly_eval_batch.restype = ctypes.c_int
        for fn in (lib.oracle_fcirc_entries, lib.oracle_polymul_coeffs, lib.oracle_bigint_mul,
                   lib.oracle_bigint_mul_school):
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(arr, ctype):
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def fcirc_entries(p: int, f: int, a, b, idx=None, threads: int | None = None) -> np.ndarray:
    """Entries ``idx`` of A*b for the f-circulant A with first row ``a`` (Definition 2).

    ``a``, ``b``: length-n sequences of residues in [0,p).  Returns uint64 array of len(idx)
    (all n entries when ``idx`` is None).
    """
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64))
    n = a.shape[0]
    assert b.shape[0] == n
    idx = np.arange(n, dtype=np.int64) if idx is None else np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    out = np.zeros(idx.shape[0], dtype=np.uint64)
    rc = lib.oracle_fcirc_entries(int(p), int(f) % int(p), _ptr(a, ctypes.c_uint64), _ptr(b, ctypes.c_uint64), n,
                                  _ptr(idx, ctypes.c_int64), idx.shape[0], _ptr(out, ctypes.c_uint64),
                                  threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_fcirc_entries: bad arguments")
    return out


def polymul_coeffs(p: int, a, b, ks=None, threads: int | None = None) -> np.ndarray:
    """Coefficients ``ks`` of a(x)*b(x) mod p, schoolbook."""
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64))
    na, nb = a.shape[0], b.shape[0]
    ks = (np.arange(na + nb - 1, dtype=np.int64) if ks is None
          else np.ascontiguousarray(np.asarray(ks, dtype=np.int64)))
    out = np.zeros(ks.shape[0], dtype=np.uint64)
    rc = lib.oracle_polymul_coeffs(int(p), _ptr(a, ctypes.c_uint64), na, _ptr(b, ctypes.c_uint64), nb,
                                   _ptr(ks, ctypes.c_int64), ks.shape[0], _ptr(out, ctypes.c_uint64),
                                   threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_polymul_coeffs: bad arguments")
    return out


# ---------------------------------------------------------------- the paper's ring
M31 = (1 << 31) - 1   # Z/pZ[sqrt 3]: u + v sqrt 3 packed as u | v << 32


def fcirc_entries_m31x2(f: int, a, b, idx=None, threads: int | None = None) -> np.ndarray:
    """Definition 2 over Z/(2^31-1)[sqrt 3]; a, b, f packed u | v << 32."""
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64))
    n = a.shape[0]
    idx = np.arange(n, dtype=np.int64) if idx is None else np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    out = np.zeros(idx.shape[0], dtype=np.uint64)
    rc = lib.oracle_fcirc_entries_m31x2(int(f), _ptr(a, ctypes.c_uint64), _ptr(b, ctypes.c_uint64), n,
                                        _ptr(idx, ctypes.c_int64), idx.shape[0], _ptr(out, ctypes.c_uint64),
                                        threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_fcirc_entries_m31x2: bad arguments")
    return out


def polymul_coeffs_m31x2(a, b, ks=None, threads: int | None = None) -> np.ndarray:
    """Schoolbook product coefficients over Z/(2^31-1)[sqrt 3] (the paper's experiment)."""
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64))
    na, nb = a.shape[0], b.shape[0]
    ks = (np.arange(na + nb - 1, dtype=np.int64) if ks is None
          else np.ascontiguousarray(np.asarray(ks, dtype=np.int64)))
    out = np.zeros(ks.shape[0], dtype=np.uint64)
    rc = lib.oracle_polymul_coeffs_m31x2(_ptr(a, ctypes.c_uint64), na, _ptr(b, ctypes.c_uint64), nb,
                                         _ptr(ks, ctypes.c_int64), ks.shape[0], _ptr(out, ctypes.c_uint64),
                                         threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_polymul_coeffs_m31x2: bad arguments")
    return out


def py_fp2_mul(x: int, y: int) -> int:
    """Python-int product in Z/(2^31-1)[sqrt 3] on packed elements (second witness, no tricks)."""
    u1, v1, u2, v2 = x & 0xFFFFFFFF, x >> 32, y & 0xFFFFFFFF, y >> 32
    return ((u1 * u2 + 3 * v1 * v2) % M31) | (((u1 * v2 + u2 * v1) % M31) << 32)


def py_fp2_pow(x: int, e: int) -> int:
    r = 1
    while e:
        if e & 1:
            r = py_fp2_mul(r, x)
        x = py_fp2_mul(x, x)
        e >>= 1
    return r


def py_fcirc_matvec_m31x2(f: int, a, b):
    """Definition 2 over Z/(2^31-1)[sqrt 3] with Python ints, for small n (witness of the C oracle)."""
    n = len(a)
    out = []
    for i in range(n):
        acc_u = acc_v = 0
        for j in range(n):
            t = py_fp2_mul(int(a[(j - i) % n]), int(b[j]))
            if j < i:
                t = py_fp2_mul(int(f), t)
            acc_u += t & 0xFFFFFFFF
            acc_v += t >> 32
        out.append((acc_u % M31) | ((acc_v % M31) << 32))
    return out


def poly_eval(p: int, c, xs, threads: int | None = None) -> np.ndarray:
    """sum_i c_i x^i mod p for each x in xs (Horner's rule).  Used for the eigen-checksum
     and Schwartz-Zippel checks of whole outputs."""
    lib = _load()
    c = np.ascontiguousarray(np.asarray(c, dtype=np.uint64))
    xs = np.ascontiguousarray(np.asarray([int(x) % int(p) for x in xs], dtype=np.uint64))
    out = np.zeros(xs.shape[0], dtype=np.uint64)
    rc = lib.oracle_poly_eval(int(p), _ptr(c, ctypes.c_uint64), c.shape[0], _ptr(xs, ctypes.c_uint64), xs.shape[0],
                              _ptr(out, ctypes.c_uint64), threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_poly_eval: bad arguments")
    return out


def eigen_thetas(p: int, n: int, w: int, count: int, seed: int) -> list[int]:
    """``count`` seeded theta with theta^n f = 1 for f = w^n: theta = w^-1 zeta_n^e."""
    import random as _random
    g = {998244353: 3, 469762049: 3, 167772161: 3, (1 << 64) - (1 << 32) + 1: 7}[int(p)]
    z = pow(g, (p - 1) // n, p)
    winv = pow(int(w), -1, p)
    rng = _random.Random(seed)
    return [winv * pow(z, rng.randrange(n), p) % p for _ in range(count)]


def eigen_check(p: int, n: int, f: int, a, b, c, thetas) -> bool:
    """sum_i c_i theta^i == (sum_j b_j theta^j)(sum_k a_k theta^-k) for every theta (theta^n f = 1)."""
    for th in thetas:
        assert pow(th, n, p) * f % p == 1
    thi = [pow(int(t), -1, p) for t in thetas]
    lhs = poly_eval(p, c, thetas)
    eb = poly_eval(p, b, thetas)
    ea = poly_eval(p, a, thi)
    return all(int(l) == int(x) * int(y) % p for l, x, y in zip(lhs, eb, ea))


def fcirc_entries_batch(p: int, f: int, a, b, idx, threads: int | None = None) -> np.ndarray:
    """``out[k, t] = (A_k b_k)_{idx[k, t]}`` for a batch (Definition 2 per instance).

    ``a``, ``b``: ``[batch, n]`` residues; ``idx``: ``[batch, m]`` entry indices per instance.
    """
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint64))
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    batch, n = a.shape
    assert b.shape == a.shape and idx.ndim == 2 and idx.shape[0] == batch
    out = np.zeros(idx.shape, dtype=np.uint64)
    rc = lib.oracle_fcirc_entries_batch(int(p), int(f) % int(p), _ptr(a, ctypes.c_uint64), _ptr(b, ctypes.c_uint64),
                                        n, batch, _ptr(idx, ctypes.c_int64), idx.shape[1],
                                        _ptr(out, ctypes.c_uint64), threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_fcirc_entries_batch: bad arguments")
    return out


def poly_eval_batch(p: int, c, xs, threads: int | None = None) -> np.ndarray:
    """``out[k, t] = sum_i c[k, i] xs[k, t]^i mod p`` (Horner) for a batch of coefficient rows."""
    lib = _load()
    c = np.ascontiguousarray(np.asarray(c, dtype=np.uint64))
    xs = np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))   # reduced mod p in the C loop
    batch, n = c.shape
    assert xs.ndim == 2 and xs.shape[0] == batch
    out = np.zeros(xs.shape, dtype=np.uint64)
    rc = lib.oracle_poly_eval_batch(int(p), _ptr(c, ctypes.c_uint64), n, batch, _ptr(xs, ctypes.c_uint64),
                                    xs.shape[1], _ptr(out, ctypes.c_uint64), threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_poly_eval_batch: bad arguments")
    return out


def eigen_thetas_batch(p: int, n: int, w: int, batch: int, count: int, seed: int) -> np.ndarray:
    """``[batch, count]`` seeded theta with theta^n f = 1 for f = w^n: theta =
    w^-1 zeta_n^e with e drawn per instance."""
    g = {998244353: 3, 469762049: 3, 167772161: 3, (1 << 64) - (1 << 32) + 1: 7}[int(p)]
    z = pow(g, (p - 1) // n, p)
    winv = pow(int(w), -1, p)
    rng = np.random.default_rng(seed)
    es = rng.integers(0, n, size=(batch, count))
    zp = {}
    out = np.zeros((batch, count), dtype=np.uint64)
    for k in range(batch):
        for t in range(count):
            e = int(es[k, t])
            if e not in zp:
                zp[e] = winv * pow(z, e, p) % p
            out[k, t] = zp[e]
    return out


def eigen_check_batch(p: int, n: int, f: int, a, b, c, thetas) -> np.ndarray:
    """Per instance: all(sum_i c_i theta^i == (sum_j b_j theta^j)(sum_k a_k theta^-k)) over its row of
    ``thetas`` (each with theta^n f = 1).  Returns a bool array [batch]."""
    thetas = np.asarray(thetas, dtype=np.uint64)
    for th in {int(t) for t in thetas.ravel()}:
        assert pow(th, n, p) * f % p == 1
    inv = {int(t): pow(int(t), -1, p) for t in set(thetas.ravel().tolist())}
    thi = np.vectorize(lambda t: inv[int(t)], otypes=[np.uint64])(thetas)
    lhs = poly_eval_batch(p, c, thetas)
    eb = poly_eval_batch(p, b, thetas)
    ea = poly_eval_batch(p, a, thi)
    ok = np.ones(thetas.shape[0], dtype=bool)
    for k in range(thetas.shape[0]):
        ok[k] = all(int(l) == int(x) * int(y) % p for l, x, y in zip(lhs[k], eb[k], ea[k]))
    return ok


def bigint_mul(x, y, school: bool = False) -> np.ndarray:
    """Full product of little-endian uint32 word arrays (independent Karatsuba)."""
    lib = _load()
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint32))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32))
    z = np.zeros(x.shape[0] + y.shape[0], dtype=np.uint32)
    fn = lib.oracle_bigint_mul_school if school else lib.oracle_bigint_mul
    rc = fn(_ptr(x, ctypes.c_uint32), x.shape[0], _ptr(y, ctypes.c_uint32), y.shape[0], _ptr(z, ctypes.c_uint32))
    if rc != 0:
        raise ValueError("oracle_bigint_mul: bad arguments")
    return z


# ----------------------------------------------------------------------------------------------
# Pure-Python witnesses (small n only)
# ----------------------------------------------------------------------------------------------

def py_fcirc_matvec(p: int, f: int, a, b) -> list[int]:
    """Definition 2 in Python ints: c_i = sum_j A[i][j] b_j, A[i][j] = a[(j-i) mod n] f^[j<i]."""
    n = len(a)
    out = []
    for i in range(n):
        s = 0
        for j in range(n):
            entry = int(a[(j - i) % n]) * (int(f) if j < i else 1)
            s += entry * int(b[j])
        out.append(s % p)
    return out


def materialize(a, f, p: int | None = None) -> list[list[int]]:
    """Build the n x n f-circulant matrix from its first row by applying Definition 2 literally.

    Rule (1): a_{i+1, j+1} = a_{i, j}.
    Rule (2): a_{i+1, 1} = a_{i, n} * f.
    (1-based in the paper; rows are built one after the other from the first row ``a``.)
    """
    n = len(a)
    rows = [[int(x) for x in a]]
    for _ in range(1, n):
        prev = rows[-1]
        new = [None] * n
        new[0] = prev[n - 1] * int(f)          # rule (2)
        for j in range(1, n):
            new[j] = prev[j - 1]               # rule (1)
        if p is not None:
            new = [v % p for v in new]
        rows.append(new)
    return rows


def matvec_dense(M, b, p: int) -> list[int]:
    """Plain dense matrix-vector product mod p (used with ``materialize``)."""
    return [sum(int(M[i][j]) * int(b[j]) for j in range(len(b))) % p for i in range(len(M))]


def alg1_recursive(p: int, f: int, a, b, sqrt_fn) -> list[int]:
    """Literal Algorithm 1 applied recursively over Z/p.

    A = [A1 A2; A2 f A1] is identified by its row a = (a1 | a2); b = (b1 | b2).
      M1 := (A1 + A2 sqrt f)(b1 sqrt f + b2)      -> sqrt(f)-circulant, row a1 + s a2
      M2 := (A1 - A2 sqrt f)(b1 sqrt f - b2)      -> (-sqrt f)-circulant, row a1 - s a2
      c1 = (M1 + M2) / (2 sqrt f),  c2 = (M1 + M2)/2 - M2
    ``sqrt_fn(f)`` returns some square root of f mod p (any sign).  Base case n = 1: c = a0 b0.
    """
    n = len(a)
    if n == 1:
        return [int(a[0]) * int(b[0]) % p]
    h = n // 2
    s = sqrt_fn(f % p)
    assert s * s % p == f % p
    a1, a2 = a[:h], a[h:]
    b1, b2 = b[:h], b[h:]
    row1 = [(int(x) + s * int(y)) % p for x, y in zip(a1, a2)]
    row2 = [(int(x) - s * int(y)) % p for x, y in zip(a1, a2)]
    v1 = [(int(x) * s + int(y)) % p for x, y in zip(b1, b2)]
    v2 = [(int(x) * s - int(y)) % p for x, y in zip(b1, b2)]
    M1 = alg1_recursive(p, s, row1, v1, sqrt_fn)
    M2 = alg1_recursive(p, (-s) % p, row2, v2, sqrt_fn)
    inv2 = pow(2, -1, p)
    inv2s = pow(2 * s % p, -1, p)
    c1 = [(m1 + m2) * inv2s % p for m1, m2 in zip(M1, M2)]
    c2 = [((m1 + m2) * inv2 - m2) % p for m1, m2 in zip(M1, M2)]
    return c1 + c2


def tonelli_shanks(x: int, p: int) -> int | None:
    """A square root of x mod the odd prime p, or None if x is a non-residue (textbook)."""
    x %= p
    if x == 0:
        return 0
    if pow(x, (p - 1) // 2, p) != 1:
        return None
    q, s = p - 1, 0
    while q % 2 == 0:
        q //= 2
        s += 1
    z = 2
    while pow(z, (p - 1) // 2, p) != p - 1:
        z += 1
    m, c, t, r = s, pow(z, q, p), pow(x, q, p), pow(x, (q + 1) // 2, p)
    while t != 1:
        i, t2 = 0, t
        while t2 != 1:
            t2 = t2 * t2 % p
            i += 1
        bb = pow(c, 1 << (m - i - 1), p)
        m, c, t, r = i, bb * bb % p, t * bb * bb % p, r * bb % p
    return r

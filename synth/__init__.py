"""synth — seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no transforms, no twist tables, no modular
products beyond the input definition f = w^n, which is how BASELINE.json's configs state
their inputs).  It only draws numbers.  Both ``tests/`` and ``bench.py`` use it; neither
``oracle/`` nor ``paper_2103_02605_b200/`` imports it.

Recipe:
  * generator ``np.random.default_rng(seed)`` (PCG64), ``seed = 2103026050 + config_index``
    unless a test passes its own;
  * draw order: w, then a, then b;
  * a, b ~ U[0, p) (uint32 for the 32-bit primes, uint64 for Goldilocks);
  * w ~ U[1, p), f = w^n mod p (so an n-th root of f exists, Theorem 1 premise),
    or f = 1 / f = p - 1 when the config names them;
  * sampled parity indices from ``default_rng(seed ^ 0xC0FFEE)`` plus the boundary indices
    {0, 1, n/2-1, n/2, n-2, n-1} where the wrap term of Definition 2 switches on.
The paper uses no public dataset (its §3.1 inputs are "polynomials with integer coefficients",
P:110-133, distribution unstated), so uniform residues stand in for them.
"""
from __future__ import annotations

import numpy as np

P998 = 998244353            # 119 * 2^23 + 1
P469 = 469762049            # 7 * 2^26 + 1
P167 = 167772161            # 5 * 2^25 + 1
GOLDILOCKS = (1 << 64) - (1 << 32) + 1
PRIMES = (P998, P469, P167, GOLDILOCKS)
BASE_SEED = 2103026050
# the paper's own ring Z/pZ[sqrt 3], p = 2^31 - 1: elements u + v sqrt 3 packed u | v << 32
M31X2 = (1 << 31) - 1


def fp2_pack(u: int, v: int) -> int:
    return (int(u) % M31X2) | ((int(v) % M31X2) << 32)


def _fp2_mul(x: int, y: int) -> int:
    """Only for the input definition f = w^n (as pow(w, n, p) for the prime fields)."""
    u1, v1, u2, v2 = x & 0xFFFFFFFF, x >> 32, y & 0xFFFFFFFF, y >> 32
    return fp2_pack(u1 * u2 + 3 * v1 * v2, u1 * v2 + u2 * v1)


def fp2_pow(x: int, e: int) -> int:
    r = 1
    while e:
        if e & 1:
            r = _fp2_mul(r, x)
        x = _fp2_mul(x, x)
        e >>= 1
    return r


def dtype_for(p: int):
    return np.uint64 if p >= (1 << 32) or p == M31X2 else np.uint32


def uniform(rng: np.random.Generator, p: int, shape) -> np.ndarray:
    """Uniform residues in [0, p) in the element dtype of p (both components for Z/p[sqrt 3])."""
    if p == M31X2:
        u = rng.integers(0, p, size=shape, dtype=np.uint64)
        v = rng.integers(0, p, size=shape, dtype=np.uint64)
        return u | (v << np.uint64(32))
    return rng.integers(0, p, size=shape, dtype=np.uint64).astype(dtype_for(p))


def edge_mix(p: int, shape, rng) -> np.ndarray:
    """Residues in [0, p) biased to the carry/borrow corner cases of the kernels' arithmetic: half of
    the entries from {0, 1, 2, p-1, p-2, 2^31 +- 1, 2^32 +- 1, 2^63, p - 2^32, ...} (those < p),
    half uniform.  No arithmetic of the method (value generation only)."""
    cand = [0, 1, 2, p - 1, p - 2, p - 3, (1 << 31) - 1, 1 << 31, (1 << 31) + 1, (1 << 32) - 1, 1 << 32,
            (1 << 32) + 1, (1 << 63) - 1, 1 << 63, (1 << 64) - (1 << 33), p - (1 << 32), p - (1 << 32) + 1,
            (p - 1) // 2, (p + 1) // 2]
    edges = np.array(sorted({c for c in cand if 0 <= c < p}), dtype=np.uint64)
    pick = edges[rng.integers(0, len(edges), size=shape)]
    unif = rng.integers(0, p, size=shape, dtype=np.uint64)
    out = np.where(rng.integers(0, 2, size=shape) == 1, pick, unif)
    return out.astype(np.uint32 if p < (1 << 32) else np.uint64)


def matvec_inputs(p: int, n: int, batch: int, seed: int, f_mode: str = "wn"):
    """Inputs of one f-circulant matvec run.

    f_mode: "wn" -> f = w^n for w ~ U[1,p);  "one" -> f = 1;  "minus_one" -> f = p - 1;
    "random" -> f ~ U[1,p) (an n-th power only with probability ~1/n; for error-path tests).
    Returns dict(p, f, w, n, batch, a[batch,n], b[batch,n]).
    """
    rng = np.random.default_rng(seed)
    w = int(rng.integers(1, p, dtype=np.uint64))
    if p == M31X2:   # w = w0 + w1 sqrt 3 (nonzero), f = w^n in Z/p[sqrt 3]
        w = fp2_pack(w, int(rng.integers(0, p, dtype=np.uint64)))
        if f_mode == "wn":
            f = fp2_pow(w, n)
        elif f_mode == "one":
            w, f = 1, 1
        elif f_mode == "minus_one":
            w, f = None, fp2_pack(p - 1, 0)
        elif f_mode == "random":
            w, f = None, w
        else:
            raise ValueError(f_mode)
    elif f_mode == "wn":
        f = pow(w, n, p)
    elif f_mode == "one":
        w, f = 1, 1
    elif f_mode == "minus_one":
        w, f = None, p - 1
    elif f_mode == "random":
        w, f = None, w
    else:
        raise ValueError(f_mode)
    a = uniform(rng, p, (batch, n))
    b = uniform(rng, p, (batch, n))
    return dict(p=p, f=f, w=w, n=n, batch=batch, a=a, b=b)


def polymul_inputs(p: int, na: int, nb: int, batch: int, seed: int):
    rng = np.random.default_rng(seed)
    a = uniform(rng, p, (batch, na))
    b = uniform(rng, p, (batch, nb))
    return dict(p=p, na=na, nb=nb, batch=batch, a=a, b=b)


def bigint_inputs(nwords: int, batch: int, seed: int):
    """Seeded uniform integers in [0, 2^(32*nwords)) as little-endian uint32 words."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 1 << 32, size=(batch, nwords), dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, 1 << 32, size=(batch, nwords), dtype=np.uint64).astype(np.uint32)
    return dict(nwords=nwords, batch=batch, x=x, y=y)


def boundary_indices(n: int):
    cand = [0, 1, n // 2 - 1, n // 2, n - 2, n - 1]
    return sorted({i for i in cand if 0 <= i < n})


def sample_indices(n: int, count: int, seed: int) -> np.ndarray:
    """``count`` seeded-random entry indices plus the boundary indices, sorted, unique."""
    rng = np.random.default_rng(seed ^ 0xC0FFEE)
    idx = set(boundary_indices(n))
    if count >= n:
        return np.arange(n, dtype=np.int64)
    idx.update(int(i) for i in rng.integers(0, n, size=count))
    return np.array(sorted(idx), dtype=np.int64)


# BASELINE.json configs (SURVEY §8 sizes table).  Index = position in BASELINE.json "configs".
CONFIGS = {
    "C1": dict(kind="matvec", p=P998, n=1 << 10, batch=1, f_mode="wn", seed=BASE_SEED + 0),
    "C2_f1": dict(kind="matvec", p=P998, n=1 << 12, batch=4096, f_mode="one", seed=BASE_SEED + 1),
    "C2_fm1": dict(kind="matvec", p=P998, n=1 << 12, batch=4096, f_mode="minus_one", seed=BASE_SEED + 1),
    "C3": dict(kind="polymul", p=P998, na=1 << 20, nb=1 << 20, batch=16, seed=BASE_SEED + 2),
    # C4 sweep: Goldilocks, n = 2^12..2^22, batch = 2^26 / n
    **{f"C4_n{L}": dict(kind="matvec", p=GOLDILOCKS, n=1 << L, batch=1 << (26 - L), f_mode="wn",
                        seed=BASE_SEED + 3) for L in range(12, 23)},
    "C5": dict(kind="bigint", nwords=1 << 17, batch=8, seed=BASE_SEED + 4),
    "S1": dict(kind="matvec", p=P998, n=1 << 20, batch=64, f_mode="wn", seed=BASE_SEED + 5),
    # NEXT-3 (Corollary 1): usual circulants (f = 1) of an order that is not a power of
    # two (n = 1000003, a prime), embedded by the library in order 2^21; batch 32
    "N3_gold": dict(kind="anyn", p=GOLDILOCKS, n=1000003, batch=32, f_mode="one", seed=BASE_SEED + 7),
    "N3_u32": dict(kind="anyn", p=P998, n=1000003, batch=32, f_mode="one", seed=BASE_SEED + 7),
    # S2 (context only): the paper's own experiment shape -- 10000 products of two
    # n-coefficient polynomials in its ring Z/(2^31-1)[sqrt 3], n = 8 .. 512
    **{f"S2_n{n}": dict(kind="polymul", p=M31X2, na=n, nb=n, batch=10000, seed=BASE_SEED + 6)
       for n in (8, 16, 32, 64, 128, 256, 512)},
}

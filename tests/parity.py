"""Parity helpers shared by the GPU tests and bench.py (test infrastructure; calls only ``oracle/``).

The rule (BASELINE.json north_star):
  * n <= 2^14: every entry of every instance against Definition 2 (O1);
  * n >  2^14: >= 1024 seeded-random entries per instance plus the boundary indices
    {0, 1, n/2-1, n/2, n-2, n-1} (where the wrap term switches on), on EVERY instance;
  * plus the eigen-checksum at >= 16 seeded theta with theta^n f = 1 on every
    instance (it covers the whole output in O(n) per theta).
Every check appends one JSON line (config, instances, entries, thetas, mismatches) to the parity
log: ``$FCIRC_PARITY_LOG``, else ``gpurun_out/parity_counts.jsonl`` when that directory exists.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FULL_MAX = 1 << 14          # every entry at or below this order
SAMPLE = 1024               # seeded entries per instance above it
THETAS = 16                 # eigen-checksum points per instance
GENERATOR = {synth.P998: 3, synth.P469: 3, synth.P167: 3, synth.GOLDILOCKS: 7}


def log_path():
    p = os.environ.get("FCIRC_PARITY_LOG")
    if p:
        return p
    d = os.path.join(ROOT, "gpurun_out")
    return os.path.join(d, "parity_counts.jsonl") if os.path.isdir(d) else None


def record(entry: dict):
    path = log_path()
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(entry) + "\n")


def root_of_f(p: int, n: int, f: int, w):
    """Some w with w^n = f for the configurations' f (the input definition, not the method): the
    drawn w for f = w^n, 1 for f = 1, a primitive 2n-th root of unity for f = p - 1."""
    if w not in (None, 0):
        return int(w)
    if f == 1:
        return 1
    if f == p - 1:
        return pow(GENERATOR[p], (p - 1) // (2 * n), p)
    raise ValueError("no known n-th root of f")


def sample_rows(n: int, batch: int, count: int, seed: int, first: int = 0) -> np.ndarray:
    """[batch, 6 + count] entry indices: the boundary indices then `count` seeded draws, per
    instance (instance k of the whole batch uses seed + first + k)."""
    bnd = np.array([0, 1, n // 2 - 1, n // 2, n - 2, n - 1], dtype=np.int64) % n
    rows = np.empty((batch, bnd.size + count), dtype=np.int64)
    for k in range(batch):
        rng = np.random.default_rng((seed + first + k) ^ 0xC0FFEE)
        rows[k, :bnd.size] = bnd
        rows[k, bnd.size:] = rng.integers(0, n, size=count)
    return rows


def check_matvec(name: str, inp: dict, c: np.ndarray, *, full: bool | None = None, sample: int = SAMPLE,
                 thetas: int = THETAS, chunk: int = 1024, seed: int = 1000) -> dict:
    """Compare the product ``c`` ([batch, n]) with the oracle on every instance; assert zero
    mismatches; return and log the coverage."""
    p, f, n, batch = inp["p"], inp["f"], inp["n"], inp["batch"]
    t0 = time.time()
    if full is None:
        full = n <= FULL_MAX
    entries = mism = 0
    first_bad = None
    for k0 in range(0, batch, chunk):
        k1 = min(batch, k0 + chunk)
        if full:
            idx = np.ascontiguousarray(np.broadcast_to(np.arange(n, dtype=np.int64), (k1 - k0, n)))
        else:
            idx = sample_rows(n, k1 - k0, sample, seed, first=k0)
        exp = oracle.fcirc_entries_batch(p, f, inp["a"][k0:k1], inp["b"][k0:k1], idx)
        got = np.take_along_axis(np.asarray(c[k0:k1]).astype(np.uint64), idx, axis=1)
        bad = np.argwhere(got != exp)
        entries += idx.size
        if bad.size:
            mism += len(bad)
            if first_bad is None:
                kk, t = bad[0]
                first_bad = (int(k0 + kk), int(idx[kk, t]), int(got[kk, t]), int(exp[kk, t]))
    th_ok = True
    if thetas and p in GENERATOR:
        w = root_of_f(p, n, f, inp.get("w"))
        for k0 in range(0, batch, chunk):
            k1 = min(batch, k0 + chunk)
            th = oracle.eigen_thetas_batch(p, n, w, k1 - k0, thetas, seed=seed + k0)
            ok = oracle.eigen_check_batch(p, n, f, inp["a"][k0:k1], inp["b"][k0:k1],
                                          np.asarray(c[k0:k1]).astype(np.uint64), th)
            if not ok.all():
                th_ok = False
                if first_bad is None:
                    first_bad = ("eigen", int(k0 + np.argmin(ok)))
    rec = {"config": name, "p": int(p), "n": int(n), "instances": int(batch), "mode": "all" if full else "sampled",
           "entries": int(entries), "thetas_per_instance": int(thetas if p in GENERATOR else 0),
           "mismatches": int(mism), "eigen_ok": bool(th_ok), "seconds": round(time.time() - t0, 2)}
    record(rec)
    assert mism == 0 and th_ok, f"{name}: {mism} mismatches / eigen {th_ok}, first {first_bad}"
    return rec


def check_polymul(name: str, inp: dict, c: np.ndarray, *, sample: int = SAMPLE, points: int = 8,
                  seed: int = 2000) -> dict:
    """Polynomial products: >= `sample` seeded coefficients + the boundary ones on every instance
    (schoolbook O2), and Schwartz-Zippel at `points` seeded x on every instance."""
    p, na, nb, batch = inp["p"], inp["na"], inp["nb"], inp["batch"]
    nc = na + nb - 1
    t0 = time.time()
    entries = mism = 0
    sz_ok = True
    for k in range(batch):
        if nc <= FULL_MAX:
            ks = np.arange(nc, dtype=np.int64)
        else:
            rng = np.random.default_rng((seed + k) ^ 0xC0FFEE)
            bnd = [0, 1, na - 1, na, nb - 1, nb, nc - 2, nc - 1]
            ks = np.unique(np.concatenate([np.array([x for x in bnd if 0 <= x < nc], dtype=np.int64),
                                           rng.integers(0, nc, size=sample)]))
        exp = oracle.polymul_coeffs(p, inp["a"][k], inp["b"][k], ks)
        got = np.asarray(c[k])[ks].astype(np.uint64)
        mism += int(np.count_nonzero(got != exp))
        entries += ks.size
        xs = [int(x) for x in np.random.default_rng(seed + 7 * k).integers(1, p, points)]
        lhs = oracle.poly_eval(p, c[k], xs)
        ea, eb = oracle.poly_eval(p, inp["a"][k], xs), oracle.poly_eval(p, inp["b"][k], xs)
        if any(int(l) != int(x) * int(y) % p for l, x, y in zip(lhs, ea, eb)):
            sz_ok = False
    rec = {"config": name, "p": int(p), "na": int(na), "nb": int(nb), "instances": int(batch),
           "entries": int(entries), "sz_points_per_instance": points, "mismatches": int(mism),
           "schwartz_zippel_ok": sz_ok, "seconds": round(time.time() - t0, 2)}
    record(rec)
    assert mism == 0 and sz_ok, rec
    return rec

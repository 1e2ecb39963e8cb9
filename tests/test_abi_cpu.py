"""CPU-side tests of the libfcirc boundary (``-m "not gpu"``): the library loads, exports every
symbol include/*.h declares, validates arguments before touching the device, and builds twist
tables that satisfy the structure of Theorem 1's proof."""
import glob
import os
import random
import re

import numpy as np
import pytest

import paper_2103_02605_b200 as fc
from synth import GOLDILOCKS, P167, P469, P998

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRIMES = [P998, P469, P167, GOLDILOCKS]
ADIC = {P998: 23, P469: 26, P167: 25, GOLDILOCKS: 32}


def _declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = fc._load()
    names = _declared_functions()
    assert {"fcirc_matvec", "fcirc_polymul", "bigint_mul", "fcirc_strerror"} <= names
    for name in sorted(names):
        assert hasattr(lib, name), name


def test_version_and_strerror():
    assert "sm_100a" in fc.version()
    for code in [0, -1, -2, -3, -4, -5, -6]:
        assert fc.strerror(code)
    assert fc.strerror(-99) == "unknown status"


def _call_matvec(p, f, n, batch, a=1, b=2, c=3):
    # fake non-null, non-overlapping device pointers: validation must fail before any device use
    lib = fc._load()
    return lib.fcirc_matvec(p, f, a << 40, b << 40, c << 40, n, batch, None)


def test_argument_validation_before_device():
    assert _call_matvec(P998, 1, 0, 1) == -1             # n < 1
    assert _call_matvec(P998, 1, 12, 1) == -1            # not a power of two
    assert _call_matvec(P998, 1, 16, 0) == -1            # batch < 1
    assert _call_matvec(P998, 1, 16, 1, a=0) == -1       # null
    assert _call_matvec(P998, 1, 16, 4, a=3, c=3) == -1  # c overlaps a
    assert _call_matvec(1000003, 1, 16, 1) == -2         # p not in the registry
    assert _call_matvec(P998, 1, 1 << 24, 1) == -4       # 2^24 does not divide p-1
    assert _call_matvec(GOLDILOCKS, 1, 1 << 25, 1) == -4  # above the maximum (2^(MMAX+KMAX) = 2^24)
    assert _call_matvec(P469, 1, 1 << 25, 1) == -4        # 2^25 | p-1 but above the 32-bit maximum 2^24
    assert _call_matvec(P998, 0, 16, 1) == -3            # f = 0: no f^-1
    assert _call_matvec(P998, P998, 16, 1) == -3         # f == 0 mod p
    # a non-residue is not a 16th power
    assert _call_matvec(P998, 3, 16, 1) == -3


@pytest.mark.parametrize("p", PRIMES)
def test_plan_table_structure(p):
    """s_{d,e}^2 = f_{d,e}; children of (d,e) carry +s and -s; s s^-1 = 1; w^n = f;
    K = n^-1 (x 2^32 for the 32-bit primes)."""
    rng = random.Random(21)
    for L in [0, 1, 2, 3, 6, 10]:
        n = 1 << L
        for f in [1, p - 1, pow(rng.randrange(1, p), n, p)]:
            if f == p - 1 and L + 1 > ADIC[p]:
                continue
            s, si, w, K = fc.plan_table(p, f, n)
            assert pow(w, n, p) == f % p
            kexp = pow(n, -1, p) * (1 if p == GOLDILOCKS else (1 << 32)) % p
            assert K == kexp
            if L == 0:
                continue
            s = [int(x) for x in s]
            si = [int(x) for x in si]
            assert s[1] * s[1] % p == f % p
            for d in range(1, L):
                for e in range(1 << d):
                    parent = s[(1 << (d - 1)) + (e >> 1)]
                    fde = parent if e % 2 == 0 else (p - parent) % p
                    assert s[(1 << d) + e] ** 2 % p == fde, (L, d, e)
            for i in range(1, n):
                assert s[i] * si[i] % p == 1


def test_plan_errors():
    with pytest.raises(fc.FcircError) as ei:
        fc.plan_table(P998, 3, 16)
    assert ei.value.code == -3
    with pytest.raises(fc.FcircError) as ei:
        fc.plan_table(P998, 1, 1 << 24)
    assert ei.value.code == -4
    with pytest.raises(fc.FcircError) as ei:
        fc.plan_table(12345, 1, 16)
    assert ei.value.code == -2


def _simulate_inplace(p, f, a, b, table):
    """Python model of the kernels' index arithmetic (in-place Algorithm 1 with the heap-indexed
    table) — host-logic check of the plan + schedule, not a product path."""
    s, si, w, K = table
    n = len(a)
    L = n.bit_length() - 1
    a = [int(x) for x in a]
    b = [int(x) for x in b]
    R = 1 << 32
    if L == 0:
        return [a[0] * b[0] % p]
    for bit in range(L - 1, -1, -1):
        for x in range(n):
            if (x >> bit) & 1:
                continue
            t = int(s[(n + x) >> (bit + 1)])
            y = x | (1 << bit)
            a[x], a[y] = (a[x] + t * a[y]) % p, (a[x] - t * a[y]) % p
            b[x], b[y] = (t * b[x] + b[y]) % p, (t * b[x] - b[y]) % p
    Rinv = 1 if p == GOLDILOCKS else pow(R, -1, p)
    m = [a[i] * b[i] * Rinv % p for i in range(n)]
    for bit in range(L):
        for x in range(n):
            if (x >> bit) & 1:
                continue
            y = x | (1 << bit)
            t = int(si[(n + x) >> (bit + 1)])
            u, v = m[x], m[y]
            m[x], m[y] = (u + v) * t % p, (u - v) % p
    return [v * K % p for v in m]


@pytest.mark.parametrize("p", PRIMES)
def test_inplace_schedule_model_matches_oracle(p):
    import oracle
    rng = random.Random(22)
    for L in range(0, 8):
        n = 1 << L
        f = pow(rng.randrange(1, p), n, p)
        a = [rng.randrange(p) for _ in range(n)]
        b = [rng.randrange(p) for _ in range(n)]
        got = _simulate_inplace(p, f, a, b, fc.plan_table(p, f, n))
        assert got == [int(x) for x in oracle.fcirc_entries(p, f, a, b)]


def test_product_package_does_not_touch_oracle():
    """The product path never imports/links the oracle."""
    pkg = os.path.join(ROOT, "paper_2103_02605_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if os.path.isfile(path) and path.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
            text = open(path).read()
            assert "import oracle" not in text and "from oracle" not in text and "liboracle" not in text, path


def test_schedule_host_only():
    """fcirc_schedule: one fused pass up to the on-chip size, then sub-problems + column levels."""
    for p in PRIMES:
        m_fused, k0 = fc.schedule(p, 1 << 10)
        assert (m_fused, k0) == (10, 0)
        M, K = fc.schedule(p, 1 << 20)
        assert M + K == 20 and 11 <= M <= 13 and K >= 7
    # the sub-problem grows only when the column passes would exceed 11 levels
    M, K = fc.schedule(P469, 1 << 24)
    assert (M, K) == (13, 11)
    with pytest.raises(fc.FcircError):
        fc.schedule(P998, 12)
    with pytest.raises(fc.FcircError):
        fc.schedule(12345, 16)


def test_circulant_any_n_validation_before_device():
    lib = fc._load()
    assert lib.fcirc_circulant_matvec(P998, 1, 2, 3, 0, 1, None) == -1        # n < 1
    assert lib.fcirc_circulant_matvec(P998, 1, 2, 3, 5, 0, None) == -1        # batch < 1
    assert lib.fcirc_circulant_matvec(P998, 0, 2, 3, 5, 1, None) == -1        # null
    assert lib.fcirc_circulant_matvec(1000003, 1, 2, 3, 5, 1, None) == -2     # p not in the registry
    assert lib.fcirc_circulant_matvec(P998, 8, 8, 8, 5, 4, None) == -1        # c overlaps a


# ---------------------------------------------------------------- the paper's ring Z/(2^31-1)[sqrt 3]

M31 = fc.M31X2


def _f2mul(x, y):
    u1, v1, u2, v2 = x & 0xFFFFFFFF, x >> 32, y & 0xFFFFFFFF, y >> 32
    return ((u1 * u2 + 3 * v1 * v2) % M31) | (((u1 * v2 + u2 * v1) % M31) << 32)


def _f2pow(x, e):
    r = 1
    while e:
        if e & 1:
            r = _f2mul(r, x)
        x = _f2mul(x, x)
        e >>= 1
    return r


def _f2neg(x):
    return ((M31 - (x & 0xFFFFFFFF)) % M31) | (((M31 - (x >> 32)) % M31) << 32)


def test_m31x2_plan_table_structure():
    """The twist table over the paper's ring: s_{d,e}^2 = f_{d,e}, children +-s,
    s s^-1 = 1, w^n = f, K = n^-1, roots of unity from the paper's generator 2 + sqrt 3."""
    rng = random.Random(31)
    for L in [0, 1, 2, 5, 9]:
        n = 1 << L
        w0 = fc.fp2_pack(rng.randrange(1, M31), rng.randrange(M31))
        for f in [1, fc.fp2_pack(M31 - 1, 0), _f2pow(w0, n)]:
            s, si, w, K = fc.plan_table(M31, f, n)
            assert _f2pow(w, n) == f
            assert K == pow(n, -1, M31)
            if L == 0:
                continue
            s = [int(x) for x in s]
            si = [int(x) for x in si]
            assert _f2mul(s[1], s[1]) == f
            for d in range(1, L):
                for e in range(1 << d):
                    parent = s[(1 << (d - 1)) + (e >> 1)]
                    fde = parent if e % 2 == 0 else _f2neg(parent)
                    assert _f2mul(s[(1 << d) + e], s[(1 << d) + e]) == fde, (L, d, e)
            for i in range(1, n):
                assert _f2mul(s[i], si[i]) == 1


def test_m31x2_premises():
    lib = fc._load()
    with pytest.raises(fc.FcircError) as ei:          # f = 0 has no inverse
        fc.plan_table(M31, 0, 16)
    assert ei.value.code == -3
    with pytest.raises(fc.FcircError) as ei:          # non-canonical packed scalar
        fc.plan_table(M31, M31, 16)
    assert ei.value.code == -1
    with pytest.raises(fc.FcircError) as ei:          # a non-square is not a 16th power:
        fc.plan_table(M31, fc.fp2_pack(1, 1), 16)     # norm(1 + sqrt 3) = -2, a non-residue (p = 7 mod 8)
    assert ei.value.code == -3
    assert fc.schedule(M31, 1 << 20) == (12, 8)
    assert lib.fcirc_matvec(M31, 1, 1, 2, 3, 1 << 25, 1, None) == -4   # above the maximum


def test_synth_edge_mix_is_canonical_and_hits_the_corners():
    """synth.edge_mix (the corner-biased parity inputs) draws canonical residues and covers the
    carry/borrow corner values it names, for every field's modulus."""
    import numpy as np
    import synth
    for p in [synth.P998, synth.P469, synth.P167, synth.GOLDILOCKS, (1 << 31) - 1]:
        x = synth.edge_mix(p, (4, 4096), np.random.default_rng(5))
        assert x.dtype == (np.uint32 if p < (1 << 32) else np.uint64)
        v = x.astype(np.uint64)
        assert int(v.max()) < p
        for corner in (0, 1, p - 1, p - 2, (1 << 31) - 1):
            if corner < p:
                assert (v == corner).any(), (p, corner)


def test_primitive_rate_and_plan_count_validation_before_device():
    """fcirc_primitive_rate rejects an unknown kind / non-positive iteration count before touching
    the device; fcirc_plan_count is host-only."""
    import ctypes
    lib = fc._load()
    ops = ctypes.c_double(0.0)
    assert lib.fcirc_primitive_rate(99, 10, ctypes.byref(ops), None, None) == -1
    assert lib.fcirc_primitive_rate(0, 0, ctypes.byref(ops), None, None) == -1
    assert lib.fcirc_primitive_rate(0, 10, None, None, None) == -1
    n, pinned = fc.plan_count()
    assert n >= 0 and 0 <= pinned <= n


def test_binding_primitive_kinds_match_header():
    """The binding's primitive-kind names map to exactly the FCIRC_PRIM_* values include/fcirc.h
    declares (bench.py's R_const / R_var probes go through these names)."""
    import re
    import paper_2103_02605_b200 as fc
    hdr = open(os.path.join(ROOT, "include", "fcirc.h")).read()
    decl = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"#define FCIRC_PRIM_(\w+) (\d+)", hdr)}
    assert decl == fc.PRIMITIVES

"""Host-side check of the Goldilocks inline-PTX carry chains in csrc/modarith.cuh.

The chains are executed by tools/ptx_carry_sim.py under the hardware carry model ptxas uses (see
its docstring) on edge and random operands and compared with Python integers.  This pins the
contracts the kernels rely on: add_c(weak, canonical) and sub_c(weak, canonical)
need one correction, sub_w(weak, weak) two, and the 128 -> 64 reduction returns the canonical
residue.  The GPU side: every kernel variant's output is compared bit for bit in tools/gold_ab.cu.
"""
import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ptx_carry_sim as sim  # noqa: E402

P = (1 << 64) - (1 << 32) + 1
M64 = (1 << 64) - 1
SRC = open(os.path.join(ROOT, "paper_2103_02605_b200", "csrc", "modarith.cuh")).read()
SRC = SRC[SRC.index("struct FieldGold {"):]

EDGE = [0, 1, 2, P - 2, P - 1, P, P + 1, M64, M64 - 1, 0xFFFFFFFF, 1 << 32, (1 << 32) + 1,
        0x8000000000000000, 0xFFFFFFFF00000000, 0xFFFFFFFEFFFFFFFF, 0x00000000FFFFFFFE]


def _pairs(rng, n=3000, a_max=M64, b_max=M64):
    for a in EDGE:
        for b in EDGE:
            if a <= a_max and b <= b_max:
                yield a, b
    for _ in range(n):
        yield rng.randint(0, a_max), rng.randint(0, b_max)
        yield rng.randint(max(0, a_max - (1 << 34)), a_max), rng.randint(max(0, b_max - (1 << 34)), b_max)


def test_add_c_predicated_weak_plus_canonical():
    """FieldGold::add_c: carry chain + predicated +EPS (setp / @p in the PTX)."""
    f = sim.helper(SRC, "add_c")
    for a, b in _pairs(random.Random(11), b_max=P - 1):
        r = f(a, b)
        assert r % P == (a + b) % P, (a, b, r)


def test_sub_c_weak_minus_canonical():
    f = sim.helper(SRC, "sub_c")
    for a, b in _pairs(random.Random(2), b_max=P - 1):
        r = f(a, b)
        assert r % P == (a - b) % P, (a, b, r)
        if a < P:
            assert r < P, "canonical minus canonical must stay canonical"


def test_sub_w_weak_minus_weak():
    f = sim.helper(SRC, "sub_w")
    for a, b in _pairs(random.Random(3)):
        r = f(a, b)
        assert r % P == (a - b) % P, (a, b, r)


@pytest.mark.parametrize("fn", ["reduce4"])
@pytest.mark.parametrize("seed", [4, 5])
def test_reduce4_canonical(seed, fn):
    f = sim.helper(SRC, fn)
    rng = random.Random(seed)
    words = [0, 1, 0xFFFFFFFF, 0xFFFFFFFE, 0x80000000]
    cases = [(a, b, c, d) for a in words for b in words for c in words for d in words]
    cases += [tuple(rng.getrandbits(32) for _ in range(4)) for _ in range(4000)]
    # full products of extreme operands
    for x in EDGE:
        for y in EDGE:
            t = x * y
            cases.append(tuple((t >> (32 * i)) & 0xFFFFFFFF for i in range(4)))
    for t0, t1, t2, t3 in cases:
        v = t0 | (t1 << 32) | (t2 << 64) | (t3 << 96)
        r = f(t0, t1, t2, t3)
        assert r == v % P, (hex(v), hex(r))


@pytest.mark.parametrize("seed", [6, 7])
def test_mont_reduce_const_times_var(seed):
    """FieldGold::mont_reduce (const x var, Montgomery R = 2^64): for T = x * s with any 64-bit x and
    s < p it returns T * 2^-64 mod p, canonical (the kernels store every table constant as s R)."""
    f = sim.helper(SRC, "mont_reduce")
    rng = random.Random(seed)
    rinv = pow(1 << 64, -1, P)
    xs = EDGE + [rng.getrandbits(64) for _ in range(1500)] + [M64 - rng.getrandbits(33) for _ in range(500)]
    ss = [0, 1, 2, P - 1, P - 2, 0xFFFFFFFF, 1 << 32, (1 << 32) + 1, 0x8000000000000000, 0xFFFFFFFF00000000,
          (1 << 32) - 1 + (1 << 63)] + [rng.randrange(P) for _ in range(40)] + [P - 1 - rng.getrandbits(33) for _ in range(20)]
    for x in xs:
        for s in ss:
            t = x * s
            r = f(*[(t >> (32 * i)) & 0xFFFFFFFF for i in range(4)])
            assert r == t * rinv % P, (hex(x), hex(s), hex(r))


@pytest.mark.parametrize("seed", [16, 17])
def test_mont_reduce_neg_is_the_negated_reduction(seed):
    """FieldGold::mont_reduce_neg (the leaves of a sub-block whose b side arrives negated from the
    column passes): -(T * 2^-64) mod p, canonical, under mont_reduce's precondition."""
    f = sim.helper(SRC, "mont_reduce_neg")
    rng = random.Random(seed)
    rinv = pow(1 << 64, -1, P)
    xs = EDGE + [rng.getrandbits(64) for _ in range(1500)] + [M64 - rng.getrandbits(33) for _ in range(500)]
    ss = [0, 1, 2, P - 1, P - 2, 0xFFFFFFFF, 1 << 32, (1 << 32) + 1, 0x8000000000000000, 0xFFFFFFFF00000000,
          (1 << 32) - 1 + (1 << 63)] + [rng.randrange(P) for _ in range(40)] + [P - 1 - rng.getrandbits(33) for _ in range(20)]
    for x in xs:
        for s in ss:
            t = x * s
            r = f(*[(t >> (32 * i)) & 0xFFFFFFFF for i in range(4)])
            assert r == (-t * rinv) % P, (hex(x), hex(s), hex(r))


@pytest.mark.parametrize("L,K,mask", [(6, 3, 0), (7, 2, 0b10011), (8, 0, 0b11000111), (5, 2, 0b111)])
def test_forward_b_negating_levels_give_popcount_signs(L, K, mask):
    """The b butterfly of a negating level (FieldGold::fwd_bn) stores y - s x for s x - y.  By linearity the
    in-place forward split of b then leaves position i of the instance times
    (-1)^(popcount(E) + popcount(x & mask)), i = E 2^M + x, when all K column levels negate and so do
    the sub-problem levels whose pair bit is in `mask` (the kernels' rule, fcirc_kernels.cuh neg_mask:
    slot bits and warp-uniform thread bits of the leaf layout): checked on a Python model of the
    in-place split over Z/p with random twiddles (the sign argument uses linearity only)."""
    rng = random.Random(5 + L)
    n, M = 1 << L, L - K
    tw = {(d, e): rng.randrange(1, P) for d in range(L) for e in range(1 << d)}
    b = [rng.randrange(P) for _ in range(n)]

    def split(negating):
        x = list(b)
        for d in range(L):
            h = n >> (d + 1)          # pair bit of level d: log2(h) = L - 1 - d
            for e in range(1 << d):
                s = tw[(d, e)]
                for j in range(h):
                    i0, i1 = e * 2 * h + j, e * 2 * h + j + h
                    t = s * x[i0] % P
                    lo = (t - x[i1]) % P
                    x[i0], x[i1] = (t + x[i1]) % P, ((-lo) % P if negating(d) else lo)
        return x
    plain = split(lambda d: False)
    # column levels d < K always negate; sub-problem level d >= K has pair bit L - 1 - d < M
    signed = split(lambda d: d < K or (mask >> (L - 1 - d)) & 1)
    for i in range(n):
        E, x = i >> M, i & ((1 << M) - 1)
        par = bin(E).count("1") + bin(x & mask).count("1")
        assert signed[i] == ((-1) ** par * plain[i]) % P, i


def test_mont_reduce_precondition_boundary():
    """The largest high word the reduction admits is p - 2 (x = 2^64 - 1, s = p - 1): still exact."""
    f = sim.helper(SRC, "mont_reduce")
    rinv = pow(1 << 64, -1, P)
    for x in [M64, M64 - 1, P, P - 1]:
        for s in [P - 1, P - 2]:
            t = x * s
            assert (t >> 64) <= P - 2
            r = f(*[(t >> (32 * i)) & 0xFFFFFFFF for i in range(4)])
            assert r == t * rinv % P


def test_canon_w_any_64_bit():
    """FieldGold::canon_w: x mod p for every 64-bit x (the leaves canonicalise one factor so that the
    Montgomery reduction's precondition holds for two weak operands)."""
    f = sim.helper(SRC, "canon_w")
    rng = random.Random(8)
    for x in EDGE + [rng.getrandbits(64) for _ in range(3000)] + [P + rng.getrandbits(32) for _ in range(500)]:
        if x > M64:
            continue
        assert f(x) == x % P, hex(x)

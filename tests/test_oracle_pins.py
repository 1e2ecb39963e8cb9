"""Pins for the CPU oracle (``-m "not gpu"``): each test checks the oracle against something
other than itself — the paper's printed 3x3 example, literal application of
Definition 2's rules (1),(2), textbook cyclic / negacyclic convolution via numpy,
closed forms, algebraic invariants, the eigen-checksum, literal Algorithm 1
with random square-root signs, SPEC hand examples, Python big ints.
"""
import json
import os
import random

import numpy as np
import pytest

import oracle
from synth import GOLDILOCKS, P167, P469, P998

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PRIMES = [P998, P469, P167, GOLDILOCKS]


def _rand(rng, p, n):
    return [rng.randrange(p) for _ in range(n)]


# ------------------------------------------------------------------ Definition 2 structure

def _load_3x3():
    rows = []
    with open(os.path.join(GOLDEN, "paper_3x3_example.txt")) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def _eval_symbol(tok, env):
    val = 1
    for part in tok.split("*"):
        val *= env[part]
    return val


@pytest.mark.parametrize("p", [P998, GOLDILOCKS])
def test_paper_3x3_example_columns(p):
    """the printed 3x3 f-circulant.  O1 with b = e_j must return column j."""
    rows = _load_3x3()
    env = {"a1": 11, "a2": 22, "a3": 33, "f": 7}
    expected = [[_eval_symbol(t, env) % p for t in r] for r in rows]
    a = [11, 22, 33]
    for j in range(3):
        e = [0, 0, 0]
        e[j] = 1
        col = oracle.fcirc_entries(p, 7, a, e)
        assert [int(x) for x in col] == [expected[i][j] for i in range(3)]
    # and the literal rule-(1),(2) materialisation reproduces the printed matrix
    assert oracle.materialize(a, 7, p) == expected


def test_materialize_vs_index_formula():
    """P:31-36 rules applied literally (row by row) vs the O1 index formula, n = 1..16."""
    rng = random.Random(1)
    for p in PRIMES:
        for n in range(1, 17):
            a, b = _rand(rng, p, n), _rand(rng, p, n)
            f = rng.randrange(1, p)
            dense = oracle.matvec_dense(oracle.materialize(a, f, p), b, p)
            got = [int(x) for x in oracle.fcirc_entries(p, f, a, b)]
            assert got == dense, (p, n)


def test_spec_hand_examples_matvec():
    with open(os.path.join(GOLDEN, "spec_hand_examples.json")) as fh:
        ex = json.load(fh)
    for case in ex["matvec"]:
        got = [int(x) for x in oracle.fcirc_entries(case["p"], case["f"], case["a"], case["b"])]
        assert got == case["c"], case["cite"]


# ------------------------------------------------------------------ textbook special cases

def test_f1_is_cyclic_correlation_numpy():
    """P:39 'a circulant 1-matrix is a usual circulant matrix': with the row convention,
    c_i = sum_k a_k b_{(i+k) mod n}; checked against numpy FFT correlation on small integers."""
    rng = np.random.default_rng(7)
    for n in [1, 2, 3, 5, 8, 16, 33, 64]:
        a = rng.integers(0, 1 << 10, n)
        b = rng.integers(0, 1 << 10, n)
        corr = np.rint(np.real(np.fft.ifft(np.conj(np.fft.fft(a)) * np.fft.fft(b)))).astype(np.int64)
        got = oracle.fcirc_entries(P998, 1, a, b).astype(np.int64)
        assert np.array_equal(got, corr % P998), n
        # cyclic convolution a (*) b = A(a~) b with a~ = (a_0, a_{n-1}, ..., a_1)
        conv = np.rint(np.real(np.fft.ifft(np.fft.fft(a) * np.fft.fft(b)))).astype(np.int64)
        at = np.concatenate([a[:1], a[1:][::-1]])
        got2 = oracle.fcirc_entries(P998, 1, at, b).astype(np.int64)
        assert np.array_equal(got2, conv % P998), n


def test_f_minus1_is_negacyclic():
    """f = -1: negacyclic convolution (mod x^n + 1) = A_{-1}(a_0, -a_{n-1}, ..., -a_1) b."""
    rng = np.random.default_rng(8)
    for p in [P998, GOLDILOCKS]:
        for n in [1, 2, 4, 7, 16, 32]:
            a = [int(x) for x in rng.integers(0, 1 << 20, n)]
            b = [int(x) for x in rng.integers(0, 1 << 20, n)]
            full = np.convolve(np.array(a, dtype=object), np.array(b, dtype=object))
            neg = [int(full[k]) - (int(full[k + n]) if k + n < len(full) else 0) for k in range(n)]
            r = [a[0] % p] + [(-x) % p for x in a[1:][::-1]]
            got = [int(x) for x in oracle.fcirc_entries(p, p - 1, r, b)]
            assert got == [v % p for v in neg], (p, n)


def test_closed_forms():
    """a = e0 -> c = b;  a = e1 -> c = (b1, ..., b_{n-1}, f b0);  b = e_j -> column j."""
    rng = random.Random(3)
    for p in [P998, GOLDILOCKS]:
        for n in [1, 2, 4, 9, 16]:
            b = _rand(rng, p, n)
            f = rng.randrange(1, p)
            e0 = [1] + [0] * (n - 1)
            assert [int(x) for x in oracle.fcirc_entries(p, f, e0, b)] == b
            if n >= 2:
                e1 = [0, 1] + [0] * (n - 2)
                assert [int(x) for x in oracle.fcirc_entries(p, f, e1, b)] == b[1:] + [f * b[0] % p]
            a = _rand(rng, p, n)
            M = oracle.materialize(a, f, p)
            for j in range(n):
                ej = [0] * n
                ej[j] = 1
                assert [int(x) for x in oracle.fcirc_entries(p, f, a, ej)] == [M[i][j] for i in range(n)]


def test_linearity_and_commutativity():
    rng = random.Random(4)
    for p in [P998, GOLDILOCKS]:
        for n in [1, 3, 8, 16]:
            f = rng.randrange(1, p)
            a, a2, b, b2 = (_rand(rng, p, n) for _ in range(4))
            lam = rng.randrange(p)
            c = lambda aa, bb: [int(x) for x in oracle.fcirc_entries(p, f, aa, bb)]
            lin_b = c(a, [(x + lam * y) % p for x, y in zip(b, b2)])
            assert lin_b == [(x + lam * y) % p for x, y in zip(c(a, b), c(a, b2))]
            lin_a = c([(x + lam * y) % p for x, y in zip(a, a2)], b)
            assert lin_a == [(x + lam * y) % p for x, y in zip(c(a, b), c(a2, b))]
            # f-circulants with the same f commute: A(a) A(a2) b = A(a2) A(a) b
            assert c(a, c(a2, b)) == c(a2, c(a, b))


def _root_of_unity(p, n):
    g = {P998: 3, P469: 3, P167: 3, GOLDILOCKS: 7}[p]
    assert (p - 1) % n == 0
    return pow(g, (p - 1) // n, p)


@pytest.mark.parametrize("p", PRIMES)
def test_eigen_checksum(p):
    """for theta^n f = 1, sum_i c_i theta^i = (sum_j b_j theta^j)(sum_k a_k theta^-k)."""
    rng = random.Random(5)
    for L in [0, 1, 2, 3, 5, 7]:
        n = 1 << L
        w = rng.randrange(1, p)
        f = pow(w, n, p)
        a, b = _rand(rng, p, n), _rand(rng, p, n)
        c = [int(x) for x in oracle.fcirc_entries(p, f, a, b)]
        z = _root_of_unity(p, n)
        winv = pow(w, -1, p)
        for e in range(min(n, 8)):
            th = winv * pow(z, e, p) % p
            assert pow(th, n, p) * f % p == 1
            thi = pow(th, -1, p)
            lhs = sum(ci * pow(th, i, p) for i, ci in enumerate(c)) % p
            rhs = (sum(bj * pow(th, j, p) for j, bj in enumerate(b)) *
                   sum(ak * pow(thi, k, p) for k, ak in enumerate(a))) % p
            assert lhs == rhs


@pytest.mark.parametrize("p", [P998, P167, GOLDILOCKS])
def test_literal_algorithm1_random_signs_equals_definition(p):
    """Theorem 1 / Algorithm 1 recursively with f' = sqrt f, f'' = -sqrt f,
    square-root signs drawn at random at every node: the result is exactly A b (Definition 2)."""
    rng = random.Random(6)

    def sqrt_fn(x):
        r = oracle.tonelli_shanks(x, p)
        assert r is not None
        return r if rng.random() < 0.5 else (-r) % p

    for L in range(0, 7):
        n = 1 << L
        for _ in range(2):
            w = rng.randrange(1, p)
            f = pow(w, n, p)
            a, b = _rand(rng, p, n), _rand(rng, p, n)
            got = oracle.alg1_recursive(p, f, a, b, sqrt_fn)
            assert got == [int(x) for x in oracle.fcirc_entries(p, f, a, b)], (p, n)


# ------------------------------------------------------------------ second witness (Python ints)

@pytest.mark.parametrize("p", PRIMES)
def test_c_oracle_vs_python_int_witness(p):
    rng = random.Random(9)
    for n in [1, 2, 5, 64, 257]:
        a, b = _rand(rng, p, n), _rand(rng, p, n)
        f = rng.randrange(1, p)
        assert [int(x) for x in oracle.fcirc_entries(p, f, a, b)] == oracle.py_fcirc_matvec(p, f, a, b)


def test_c_oracle_accumulator_extremes():
    """All-(p-1) inputs stress the 192-bit accumulator (Goldilocks products are ~2^128)."""
    for p in [GOLDILOCKS, P998]:
        for n in [1024, 4096]:
            a = [p - 1] * n
            b = [p - 1] * n
            f = p - 1
            idx = [0, 1, n // 2, n - 1]
            got = [int(x) for x in oracle.fcirc_entries(p, f, a, b, idx)]
            # closed form: c_i = (n - i) (p-1)^2 + f i (p-1)^2
            exp = [((n - i) * (p - 1) ** 2 + f * i * (p - 1) ** 2) % p for i in idx]
            assert got == exp


def test_threads_do_not_change_results():
    rng = np.random.default_rng(10)
    n = 4096
    a = rng.integers(0, GOLDILOCKS, n, dtype=np.uint64)
    b = rng.integers(0, GOLDILOCKS, n, dtype=np.uint64)
    idx = rng.integers(0, n, 97)
    r1 = oracle.fcirc_entries(GOLDILOCKS, 12345, a, b, idx, threads=1)
    r8 = oracle.fcirc_entries(GOLDILOCKS, 12345, a, b, idx, threads=8)
    assert np.array_equal(r1, r8)


def test_bad_arguments_raise():
    with pytest.raises(ValueError):
        oracle.fcirc_entries(P998, 1, [1, 2], [3, 4], idx=[2])


# ------------------------------------------------------------------ polynomial products

def test_spec_hand_examples_polymul_bigint():
    with open(os.path.join(GOLDEN, "spec_hand_examples.json")) as fh:
        ex = json.load(fh)
    for case in ex["polymul"]:
        got = [int(x) for x in oracle.polymul_coeffs(case["p"], case["a"], case["b"])]
        assert got == case["c"], case["cite"]
    for case in ex["bigint"]:
        x, y = case["x"], case["y"]
        xw = _to_words(x) or [0]
        yw = _to_words(y) or [0]
        z = oracle.bigint_mul(xw, yw)
        assert _from_words(z) == case["z"], case["cite"]


def test_polymul_vs_numpy_convolve():
    rng = np.random.default_rng(11)
    for na, nb in [(1, 1), (3, 2), (17, 33), (200, 150)]:
        for p in [P998, GOLDILOCKS]:
            a = rng.integers(0, p, na, dtype=np.uint64)
            b = rng.integers(0, p, nb, dtype=np.uint64)
            ref = np.convolve(a.astype(object), b.astype(object))
            got = oracle.polymul_coeffs(p, a, b)
            assert [int(x) for x in got] == [int(v) % p for v in ref]


def test_polymul_schwartz_zippel():
    """C(x0) = A(x0) B(x0) mod p at seeded points (length law: na + nb - 1 coefficients)."""
    rng = np.random.default_rng(12)
    p = P998
    a = rng.integers(0, p, 3000, dtype=np.uint64)
    b = rng.integers(0, p, 2000, dtype=np.uint64)
    c = oracle.polymul_coeffs(p, a, b)
    assert c.shape[0] == 3000 + 2000 - 1

    def ev(coef, x0):
        acc = 0
        for v in reversed([int(t) for t in coef]):
            acc = (acc * x0 + v) % p
        return acc

    for x0 in [int(t) for t in rng.integers(1, p, 8)]:
        assert ev(c, x0) == ev(a, x0) * ev(b, x0) % p


# ------------------------------------------------------------------ big integers

def _to_words(v):
    out = []
    while v:
        out.append(v & 0xFFFFFFFF)
        v >>= 32
    return out


def _from_words(ws):
    v = 0
    for i, w in enumerate(ws):
        v |= int(w) << (32 * i)
    return v


def test_karatsuba_vs_python_int_and_school():
    rng = random.Random(13)
    for nx, ny in [(1, 1), (1, 7), (31, 33), (64, 64), (100, 37), (257, 1000), (1 << 12, 1 << 12)]:
        x = [rng.randrange(1 << 32) for _ in range(nx)]
        y = [rng.randrange(1 << 32) for _ in range(ny)]
        if nx > 3:
            x[-1] = 0xFFFFFFFF
            x[1] = 0xFFFFFFFF
        z = oracle.bigint_mul(x, y)
        assert _from_words(z) == _from_words(x) * _from_words(y), (nx, ny)
        if nx * ny <= 1 << 20:
            assert np.array_equal(z, oracle.bigint_mul(x, y, school=True))


def test_karatsuba_all_ones():
    for n in [33, 64, 65, 1000]:
        x = [0xFFFFFFFF] * n
        z = oracle.bigint_mul(x, x)
        assert _from_words(z) == ((1 << (32 * n)) - 1) ** 2


def test_oracle_header_says_test_infrastructure():
    here = os.path.dirname(oracle.__file__)
    for name in ("__init__.py", "oracle.c"):
        with open(os.path.join(here, name)) as fh:
            assert "TEST INFRASTRUCTURE" in fh.read(4000)


def test_poly_eval_vs_python_horner_and_closed_forms():
    rng = random.Random(14)
    for p in [P998, GOLDILOCKS]:
        c = [rng.randrange(p) for _ in range(300)]
        xs = [0, 1, p - 1, rng.randrange(p), rng.randrange(p)]
        got = [int(v) for v in oracle.poly_eval(p, c, xs)]
        assert got[0] == c[0]
        assert got[1] == sum(c) % p
        assert got[2] == sum(ci * (-1) ** i for i, ci in enumerate(c)) % p
        for x, g in zip(xs[3:], got[3:]):
            assert g == sum(ci * pow(x, i, p) for i, ci in enumerate(c)) % p


def test_eigen_check_detects_a_single_corrupted_entry():
    rng = random.Random(15)
    p, n = P998, 64
    w = rng.randrange(1, p)
    f = pow(w, n, p)
    a = [rng.randrange(p) for _ in range(n)]
    b = [rng.randrange(p) for _ in range(n)]
    c = [int(x) for x in oracle.fcirc_entries(p, f, a, b)]
    th = oracle.eigen_thetas(p, n, w, 4, seed=1)
    assert oracle.eigen_check(p, n, f, a, b, c, th)
    c[17] = (c[17] + 1) % p
    assert not oracle.eigen_check(p, n, f, a, b, c, th)


def test_poly_eval_batch_vs_power_sums_and_closed_forms():
    """Batched Horner (oracle_poly_eval_batch): per-instance rows and points.  Pinned by
    x = 0 -> c_0, x = 1 -> sum c, x = -1 -> alternating sum, the geometric closed form
    sum_{i<n} x^i = (x^n - 1)/(x - 1) on an all-ones row, and power sums with Python ints."""
    rng = random.Random(16)
    for p in [P998, GOLDILOCKS]:
        batch, n = 5, 257
        c = np.array([[rng.randrange(p) for _ in range(n)] for _ in range(batch)], dtype=np.uint64)
        c[3, :] = 1
        xs = np.array([[0, 1, p - 1, rng.randrange(2, p)] for _ in range(batch)], dtype=np.uint64)
        got = oracle.poly_eval_batch(p, c, xs)
        for k in range(batch):
            row = [int(v) for v in c[k]]
            assert int(got[k, 0]) == row[0]
            assert int(got[k, 1]) == sum(row) % p
            assert int(got[k, 2]) == sum(ci * (-1) ** i for i, ci in enumerate(row)) % p
            x = int(xs[k, 3])
            if k == 3:
                assert int(got[k, 3]) == (pow(x, n, p) - 1) * pow(x - 1, -1, p) % p
            assert int(got[k, 3]) == sum(ci * pow(x, i, p) for i, ci in enumerate(row)) % p


def test_fcirc_entries_batch_indexing_and_closed_forms():
    """The batched entry oracle uses instance k's own a, b and index row: pinned per instance by
    the closed forms a = e_0 -> c = b and a = e_1 -> c = (b_1, .., b_{n-1}, f b_0) (Definition 2,
    P:29-37) placed at different instances of one batch, and by the Python-int witness."""
    rng = random.Random(17)
    for p in [P998, GOLDILOCKS]:
        n, batch = 24, 4
        f = rng.randrange(1, p)
        a = np.array([[rng.randrange(p) for _ in range(n)] for _ in range(batch)], dtype=np.uint64)
        b = np.array([[rng.randrange(p) for _ in range(n)] for _ in range(batch)], dtype=np.uint64)
        a[1, :] = 0
        a[1, 0] = 1
        a[2, :] = 0
        a[2, 1] = 1
        idx = np.array([rng.sample(range(n), 9) for _ in range(batch)], dtype=np.int64)
        got = oracle.fcirc_entries_batch(p, f, a, b, idx)
        bl = [[int(v) for v in row] for row in b]
        shift = bl[2][1:] + [f * bl[2][0] % p]
        for t in range(9):
            assert int(got[1, t]) == bl[1][idx[1, t]]
            assert int(got[2, t]) == shift[idx[2, t]]
        for k in (0, 3):
            full = oracle.py_fcirc_matvec(p, f, [int(v) for v in a[k]], bl[k])
            assert [int(v) for v in got[k]] == [full[i] for i in idx[k]]


def test_eigen_check_batch_flags_only_the_corrupted_instance():
    rng = random.Random(18)
    for p in [P998, GOLDILOCKS]:
        n, batch = 32, 6
        w = rng.randrange(1, p)
        f = pow(w, n, p)
        a = np.array([[rng.randrange(p) for _ in range(n)] for _ in range(batch)], dtype=np.uint64)
        b = np.array([[rng.randrange(p) for _ in range(n)] for _ in range(batch)], dtype=np.uint64)
        c = np.stack([oracle.fcirc_entries(p, f, a[k], b[k]) for k in range(batch)])
        th = oracle.eigen_thetas_batch(p, n, w, batch, 16, seed=3)
        for k in range(batch):
            for t in th[k]:
                assert pow(int(t), n, p) * f % p == 1
        assert oracle.eigen_check_batch(p, n, f, a, b, c, th).all()
        c[4, 9] = (int(c[4, 9]) + 1) % p
        ok = oracle.eigen_check_batch(p, n, f, a, b, c, th)
        assert not ok[4] and ok[[0, 1, 2, 3, 5]].all()


def test_corollary1_embedding_any_n():
    """Corollary 1: for non-power-of-two n, the order-N circulant with row
    a' = (a_1..a_n, 0..0, a_2..a_n) times b' = (b, 0..0) has A b as its first n entries -- with the
    paper's N = 2^{d+1} (2^d the smallest power of two > n) and with the smallest power of two
    N >= 2n - 1 that libfcirc uses (reading R10).  Oracle = Definition 2 at both orders."""
    import oracle
    rng = random.Random(102)
    p = P998
    for n in list(range(1, 41)) + [63, 65, 100]:
        a = [rng.randrange(p) for _ in range(n)]
        b = [rng.randrange(p) for _ in range(n)]
        ref = [int(v) for v in oracle.fcirc_entries(p, 1, a, b)]
        d = 0
        while (1 << d) <= n:
            d += 1
        paper_N = 1 << (d + 1)
        min_N = 1
        while min_N < 2 * n - 1:
            min_N <<= 1
        for N in {paper_N, min_N}:
            a2 = a + [0] * (N - 2 * n + 1) + a[1:]
            b2 = b + [0] * (N - n)
            assert len(a2) == N and len(b2) == N
            got = [int(v) for v in oracle.fcirc_entries(p, 1, a2, b2)][:n]
            assert got == ref, (n, N)


# ---------------------------------------------------------------- the paper's ring

def test_m31x2_paper_generator_and_ring():
    """in Z/pZ[sqrt 3] (p = 2^31 - 1, 3 a non-residue) 2 + sqrt 3 generates the roots of unity:
    its order is p + 1 = 2^31; sqrt 3 squares to 3."""
    import oracle
    M = oracle.M31
    assert pow(3, (M - 1) // 2, M) == M - 1                      # 3 is a non-residue mod p
    g = 2 | (1 << 32)
    assert oracle.py_fp2_pow(g, 1 << 31) == 1
    assert oracle.py_fp2_pow(g, 1 << 30) == M - 1                # -1: order exactly 2^31
    assert oracle.py_fp2_mul(1 << 32, 1 << 32) == 3


def test_m31x2_oracle_vs_python_witness_and_3x3():
    """C oracle over Z/(2^31-1)[sqrt 3] = the Python-int witness; the 3x3 example's columns."""
    import oracle
    M = oracle.M31
    rng = random.Random(77)
    pk = lambda u, v: (u % M) | ((v % M) << 32)  # noqa: E731
    for n in [1, 2, 3, 5, 8, 12]:
        a = [pk(rng.randrange(M), rng.randrange(M)) for _ in range(n)]
        b = [pk(rng.randrange(M), rng.randrange(M)) for _ in range(n)]
        f = pk(rng.randrange(1, M), rng.randrange(M))
        assert [int(x) for x in oracle.fcirc_entries_m31x2(f, a, b)] == oracle.py_fcirc_matvec_m31x2(f, a, b)
    a = [pk(11, 1), pk(22, 2), pk(33, 3)]
    f = pk(7, 5)
    af = [oracle.py_fp2_mul(f, x) for x in a]
    cols = [[a[0], af[2], af[1]], [a[1], a[0], af[2]], [a[2], a[1], a[0]]]   # column j of P:42-44
    for j in range(3):
        e = [0, 0, 0]
        e[j] = 1
        assert [int(x) for x in oracle.fcirc_entries_m31x2(f, a, e)] == cols[j]


def test_m31x2_polymul_oracle_vs_python():
    import oracle
    M = oracle.M31
    rng = random.Random(78)
    pk = lambda u, v: (u % M) | ((v % M) << 32)  # noqa: E731
    a = [pk(rng.randrange(M), rng.randrange(M)) for _ in range(9)]
    b = [pk(rng.randrange(M), rng.randrange(M)) for _ in range(6)]
    exp = []
    for k in range(14):
        au = av = 0
        for i in range(max(0, k - 5), min(k, 8) + 1):
            t = oracle.py_fp2_mul(a[i], b[k - i])
            au += t & 0xFFFFFFFF
            av += t >> 32
        exp.append((au % M) | ((av % M) << 32))
    assert [int(x) for x in oracle.polymul_coeffs_m31x2(a, b)] == exp

"""GPU parity: the CUDA path (through the C ABI via the thin binding) against the CPU oracle,
element by element, bit-exact (integer work).

Coverage rules:
  * n <= 2^14: every entry of every instance (small batches; several tiles + ragged batch);
  * n >  2^14 and BASELINE.json full sizes: >= 1024 seeded-random entries per checked instance
    plus the boundary indices {0, 1, n/2-1, n/2, n-2, n-1}, and the eigen-checksum
     on whole outputs;
  * polymul: sampled coefficients + Schwartz-Zippel; bigint: the full product vs Python ints and
    the oracle's Karatsuba.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import GOLDILOCKS, P167, P469, P998

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2103_02605_b200 as fc  # noqa: E402

PRIMES = [P998, P469, P167, GOLDILOCKS]
ADIC = {P998: 23, P469: 26, P167: 25, GOLDILOCKS: 32}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


def _dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _host(t) -> np.ndarray:
    return t.cpu().numpy()


def run_matvec(inp):
    a, b = _dev(inp["a"]), _dev(inp["b"])
    c = fc.matvec(a, b, inp["f"], inp["p"])
    torch.cuda.synchronize()
    return _host(c)


def check_full(inp, c, instances=None):
    p, f = inp["p"], inp["f"]
    for k in (range(inp["batch"]) if instances is None else instances):
        exp = oracle.fcirc_entries(p, f, inp["a"][k], inp["b"][k])
        got = c[k].astype(np.uint64)
        bad = np.nonzero(got != exp)[0]
        assert bad.size == 0, f"instance {k}: {bad.size} mismatches, first at {bad[0]}: got {got[bad[0]]} exp {exp[bad[0]]}"


def check_sampled(inp, c, instances, count=1024, thetas=4):
    p, f, n = inp["p"], inp["f"], inp["n"]
    for k in instances:
        idx = synth.sample_indices(n, count, seed=1000 + k)
        exp = oracle.fcirc_entries(p, f, inp["a"][k], inp["b"][k], idx)
        got = c[k][idx].astype(np.uint64)
        bad = np.nonzero(got != exp)[0]
        assert bad.size == 0, f"instance {k}: {bad.size} mismatches, first idx {idx[bad[0]]}"
        if thetas and inp.get("w"):
            th = oracle.eigen_thetas(p, n, inp["w"], thetas, seed=k)
            assert oracle.eigen_check(p, n, f, inp["a"][k], inp["b"][k], c[k], th), f"eigen-checksum, instance {k}"


# ---------------------------------------------------------------------------------- fused path

@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("f_mode", ["wn", "one", "minus_one"])
def test_matvec_all_entries_small(p, f_mode):
    """n = 2^0 .. 2^14, every entry; batch 3 (ragged against the instances-per-CTA packing)."""
    for L in range(0, 15):
        if f_mode == "minus_one" and L + 1 > ADIC[p]:
            continue
        batch = 3 if L <= 12 else 2
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=100 + L, f_mode=f_mode)
        c = run_matvec(inp)
        check_full(inp, c)


@pytest.mark.parametrize("p", [P998, GOLDILOCKS])
def test_matvec_many_instances_small_n(p):
    """Many instances per launch (grid of several waves, ragged last CTA)."""
    for L, batch in [(1, 1001), (4, 777), (7, 333), (10, 149)]:
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=7 + L)
        c = run_matvec(inp)
        check_full(inp, c, instances=[0, 1, batch // 2, batch - 2, batch - 1])
        th_ok = all(oracle.eigen_check(p, 1 << L, inp["f"], inp["a"][k], inp["b"][k], c[k],
                                       oracle.eigen_thetas(p, 1 << L, inp["w"], 2, seed=k)) for k in range(batch))
        assert th_ok


def test_matvec_extreme_values():
    """All inputs p-1 (largest residues) and zeros, Goldilocks and 32-bit, fused and multi-pass."""
    for p in [P998, GOLDILOCKS]:
        for L in [3, 11, 12, 16]:
            n = 1 << L
            dt = np.uint64 if p == GOLDILOCKS else np.uint32
            for val in [p - 1, 0, 1]:
                inp = dict(p=p, n=n, batch=1, f=p - 1, w=None,
                           a=np.full((1, n), val, dtype=dt), b=np.full((1, n), p - 1, dtype=dt))
                c = run_matvec(inp)
                if n <= 1 << 12:
                    check_full(inp, c)
                else:
                    check_sampled(inp, c, [0], count=256, thetas=0)


@pytest.mark.parametrize("p", PRIMES)
def test_matvec_edge_value_mix(p):
    """Inputs biased to the carry / borrow / canonicalisation corners (synth.edge_mix: p-1, p-2,
    2^32 +- 1, 2^63, p - 2^32, ...): every entry through the fused (n <= 2^12) and the three-pass
    (2^13) schedules, sampled entries + checksum at 2^16."""
    rng = np.random.default_rng(4242 + p % 1000)
    for L in [10, 12, 13, 16]:
        n = 1 << L
        w = int(rng.integers(1, p, dtype=np.uint64))
        inp = dict(p=p, n=n, batch=2, f=pow(w, n, p), w=w,
                   a=synth.edge_mix(p, (2, n), rng), b=synth.edge_mix(p, (2, n), rng))
        c = run_matvec(inp)
        if L <= 13:
            check_full(inp, c)
        else:
            check_sampled(inp, c, [0, 1], count=512, thetas=2)


# ---------------------------------------------------------------------------------- multi-pass

@pytest.mark.parametrize("p", PRIMES)
def test_matvec_multipass_sampled(p):
    """n = 2^13 .. the maximum (2^23, or 2^24 for the primes with 2-adicity > 23): three-pass
    schedule, sampled entries + checksum."""
    top = {P998: 23, P469: 24, P167: 24, GOLDILOCKS: 24}[p]
    for L in range(13, top + 1):
        batch = 3 if L <= 18 else 1
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=200 + L)
        c = run_matvec(inp)
        check_sampled(inp, c, range(batch), count=1024 if L <= 20 else (512 if L <= 22 else 256), thetas=2)


def test_matvec_multipass_full_entries_2pow15():
    for p in [P998, GOLDILOCKS]:
        inp = synth.matvec_inputs(p, 1 << 15, 2, seed=33)
        c = run_matvec(inp)
        check_full(inp, c)


def test_matvec_chunking_ragged(monkeypatch):
    """Batch not a multiple of the L2 chunk: instances in the last, short chunk are right."""
    inp = synth.matvec_inputs(GOLDILOCKS, 1 << 16, 7, seed=44)
    c = run_matvec(inp)
    check_sampled(inp, c, range(7), count=256, thetas=1)


# ---------------------------------------------------------------------------------- BASELINE configs

def test_config_C1():
    inp = synth.matvec_inputs(**{k: v for k, v in synth.CONFIGS["C1"].items() if k != "kind"})
    c = run_matvec(inp)
    check_full(inp, c)


@pytest.mark.parametrize("name", ["C2_f1", "C2_fm1"])
def test_config_C2(name):
    cfg = {k: v for k, v in synth.CONFIGS[name].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    rng = np.random.default_rng(5)
    check_full(inp, c, instances=sorted({0, 4095, *rng.integers(0, 4096, 30).tolist()}))
    # every instance: eigen-checksum (f = 1 -> theta^n = 1; f = -1 -> theta^n = -1)
    p, n, f = inp["p"], inp["n"], inp["f"]
    g = 3
    z2n = pow(g, (p - 1) // (2 * n), p)
    th = [1, pow(g, (p - 1) // n, p)] if f == 1 else [pow(z2n, -1, p), pow(z2n, -3, p)]
    for k in range(inp["batch"]):
        assert oracle.eigen_check(p, n, f, inp["a"][k], inp["b"][k], c[k], th), k


@pytest.mark.parametrize("L", list(range(12, 23)))
def test_config_C4_goldilocks_sweep(L):
    cfg = {k: v for k, v in synth.CONFIGS[f"C4_n{L}"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    batch = inp["batch"]
    ks = sorted({0, 1, batch // 2, batch - 1})
    if L <= 14:
        check_full(inp, c, instances=ks[:2])
    check_sampled(inp, c, ks, count=1024, thetas=2)


def test_config_S1():
    cfg = {k: v for k, v in synth.CONFIGS["S1"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_sampled(inp, c, [0, 1, 31, 62, 63], count=1024, thetas=2)


# ---------------------------------------------------------------------------------- host entry

def test_matvec_host_matches_device():
    for p, L, batch in [(GOLDILOCKS, 11, 5), (P998, 16, 9), (GOLDILOCKS, 20, 3)]:
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=55 + L)
        c_host = fc.matvec_host(inp["a"], inp["b"], inp["f"], p)
        c_dev = run_matvec(inp)
        assert np.array_equal(c_host, c_dev)
        check_sampled(inp, c_host, [0, batch - 1], count=256, thetas=1)


def test_errors_through_binding():
    a = torch.zeros((2, 16), dtype=torch.int64, device="cuda")
    with pytest.raises(fc.FcircError) as ei:
        fc.matvec(a, a.clone(), 7, GOLDILOCKS)  # 7 generates (Z/p)^*: not a square
    assert ei.value.code in (-3,)
    with pytest.raises(fc.FcircError) as ei:
        fc.matvec(a[:, :12].contiguous(), a[:, :12].contiguous(), 1, GOLDILOCKS)
    assert ei.value.code == -1
    with pytest.raises(fc.FcircError) as ei:
        fc.matvec(a, a, 1, GOLDILOCKS, out=a)
    assert ei.value.code == -1


def test_nondefault_stream_and_repeatability():
    inp = synth.matvec_inputs(GOLDILOCKS, 1 << 14, 4, seed=66)
    a, b = _dev(inp["a"]), _dev(inp["b"])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        c1 = fc.matvec(a, b, inp["f"], GOLDILOCKS)
        c2 = fc.matvec(a, b, inp["f"], GOLDILOCKS)
    s.synchronize()
    assert torch.equal(c1, c2)
    check_sampled(inp, _host(c1), [0, 3], count=512, thetas=1)


# ---------------------------------------------------------------------------------- polymul

@pytest.mark.parametrize("p", [P998, GOLDILOCKS])
def test_polymul_small_full(p):
    rng = np.random.default_rng(77)
    # fused single pass (L <= 2^MMAX) and multi-pass (embedding fused into the first column pass,
    # truncation into the last); degenerate one-coefficient operands on either side
    for na, nb, batch in [(1, 1, 2), (2, 3, 2), (17, 33, 3), (1000, 24, 2), (4096, 4096, 2), (5000, 3000, 1),
                          (1, 9000, 2), (9000, 1, 2), (10000, 7000, 2), (20000, 45000, 1)]:
        inp = synth.polymul_inputs(p, na, nb, batch, seed=int(rng.integers(1 << 30)))
        c = fc.polymul(_dev(inp["a"]), _dev(inp["b"]), p)
        c = _host(c)
        for k in range(batch):
            exp = oracle.polymul_coeffs(p, inp["a"][k], inp["b"][k])
            assert np.array_equal(c[k].astype(np.uint64), exp), (na, nb, k)


@pytest.mark.parametrize("p", [P998, GOLDILOCKS])
def test_polymul_edge_value_mix(p):
    """Polynomial products on corner-biased coefficients (synth.edge_mix), fused and multi-pass."""
    rng = np.random.default_rng(99)
    for na, nb in [(100, 77), (3000, 2000), (9000, 7000)]:
        a, b = synth.edge_mix(p, (2, na), rng), synth.edge_mix(p, (2, nb), rng)
        c = _host(fc.polymul(_dev(a), _dev(b), p))
        for k in range(2):
            assert np.array_equal(c[k].astype(np.uint64), oracle.polymul_coeffs(p, a[k], b[k])), (na, nb, k)


def test_config_C3_polymul():
    cfg = synth.CONFIGS["C3"]
    inp = synth.polymul_inputs(cfg["p"], cfg["na"], cfg["nb"], cfg["batch"], cfg["seed"])
    c = _host(fc.polymul(_dev(inp["a"]), _dev(inp["b"]), cfg["p"]))
    p, nc = cfg["p"], cfg["na"] + cfg["nb"] - 1
    assert c.shape == (cfg["batch"], nc)
    for k in [0, 7, 15]:
        ks = np.unique(np.concatenate([synth.sample_indices(nc, 1024, seed=k),
                                       [0, 1, (1 << 20) - 1, 1 << 20, nc - 1]]))
        exp = oracle.polymul_coeffs(p, inp["a"][k], inp["b"][k], ks)
        assert np.array_equal(c[k][ks].astype(np.uint64), exp), k
        xs = [int(x) for x in np.random.default_rng(k).integers(1, p, 8)]
        assert np.array_equal(oracle.poly_eval(p, c[k], xs),
                              (oracle.poly_eval(p, inp["a"][k], xs).astype(object) *
                               oracle.poly_eval(p, inp["b"][k], xs).astype(object) % p).astype(np.uint64))


# ---------------------------------------------------------------------------------- bigint

def _to_int(words):
    return int.from_bytes(np.ascontiguousarray(words, dtype="<u4").tobytes(), "little")


def test_bigint_small():
    rng = np.random.default_rng(88)
    for nx, ny, batch in [(1, 1, 3), (1, 5, 2), (7, 3, 2), (64, 64, 2), (1000, 777, 2), (4096, 4096, 1)]:
        inp = synth.bigint_inputs(max(nx, ny), batch, seed=int(rng.integers(1 << 30)))
        x = np.ascontiguousarray(inp["x"][:, :nx])
        y = np.ascontiguousarray(inp["y"][:, :ny])
        z = _host(fc.bigint_mul(_dev(x), _dev(y)))
        for k in range(batch):
            assert _to_int(z[k]) == _to_int(x[k]) * _to_int(y[k]), (nx, ny, k)


def test_bigint_edge_values():
    # all-ones operands: (2^32m - 1)^2 has a run of 0xFFFF digits, so the carry crosses many
    # 2048-digit segments of the carry scan (nx = 5000: 20000 digits, 10 segments)
    for nx in [1, 2, 33, 1025, 5000]:
        ones = np.full((1, nx), 0xFFFFFFFF, dtype=np.uint32)
        zeros = np.zeros((1, nx), dtype=np.uint32)
        one = np.zeros((1, nx), dtype=np.uint32)
        one[0, 0] = 1
        for x, y in [(ones, ones), (zeros, ones), (one, ones)]:
            z = _host(fc.bigint_mul(_dev(x), _dev(y)))
            assert _to_int(z[0]) == _to_int(x[0]) * _to_int(y[0])
    z = _host(fc.bigint_mul(_dev(np.array([[999]], dtype=np.uint32)), _dev(np.array([[999]], dtype=np.uint32))))
    assert _to_int(z[0]) == 998001


def test_config_C5_bigint():
    cfg = synth.CONFIGS["C5"]
    inp = synth.bigint_inputs(cfg["nwords"], cfg["batch"], cfg["seed"])
    z = _host(fc.bigint_mul(_dev(inp["x"]), _dev(inp["y"])))
    for k in range(cfg["batch"]):
        assert _to_int(z[k]) == _to_int(inp["x"][k]) * _to_int(inp["y"][k]), k
    # and against the oracle's independent Karatsuba, word for word
    assert np.array_equal(z[0], oracle.bigint_mul(inp["x"][0], inp["y"][0]))


# ---------------------------------------------------------------------------------- runtime

def test_plan_cache_eviction_many_f():
    """More distinct (p, f, n) plans than the cache keeps (64): evicted plans are rebuilt and every
    result stays exact (no stale or freed twist table is used)."""
    rng = np.random.default_rng(123)
    for i in range(80):
        p = P998 if i % 2 else GOLDILOCKS
        inp = synth.matvec_inputs(p, 1 << 9, 2, seed=int(rng.integers(1 << 30)))
        c = run_matvec(inp)
        if i % 10 == 0 or i > 70:
            check_full(inp, c)


def test_concurrent_host_threads_and_streams():
    """Two host threads, each on its own stream, issue products concurrently (plan cache and
    workspace pool are shared and mutex-guarded)."""
    import threading
    results, errors = {}, []

    def work(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for j in range(6):
                    p = GOLDILOCKS if (tid + j) % 2 else P998
                    inp = synth.matvec_inputs(p, 1 << (14 + j % 3), 2, seed=1000 * tid + j)
                    a, b = _dev(inp["a"]), _dev(inp["b"])
                    c = fc.matvec(a, b, inp["f"], p, stream=s)
                    s.synchronize()
                    results[(tid, j)] = (inp, _host(c))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for (tid, j), (inp, c) in results.items():
        check_sampled(inp, c, [0, 1], count=256, thetas=1)


def test_check_inputs_mode_rejects_noncanonical():
    """FCIRC_CHECK_INPUTS=1 (debug mode): an input >= p is reported as FCIRC_EINVAL instead of
    producing a silently wrong product.  Runs in a subprocess (the knob is read once)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, paper_2103_02605_b200 as fc, synth
inp = synth.matvec_inputs(synth.P998, 1 << 12, 2, seed=5)
a = torch.from_numpy(inp["a"]).cuda(); b = torch.from_numpy(inp["b"]).cuda()
fc.matvec(a, b, inp["f"], synth.P998)                       # canonical: accepted
bad = inp["a"].copy(); bad[1, 77] = synth.P998              # == p: not canonical
a = torch.from_numpy(bad).cuda()
try:
    fc.matvec(a, b, inp["f"], synth.P998)
    print("accepted")
except fc.FcircError as e:
    print("rejected", e.code)
'''
    env = dict(os.environ, FCIRC_CHECK_INPUTS="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "rejected -1" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("p", [P998, GOLDILOCKS])
def test_circulant_any_n_corollary1(p):
    """fcirc_circulant_matvec (Corollary 1): usual circulant of any order n, every entry
    against Definition 2 with f = 1 -- fused (N <= 2^12) and multi-pass embeddings, powers of two."""
    for n, batch in [(1, 3), (3, 2), (5, 2), (7, 3), (100, 2), (1000, 2), (1024, 2), (3000, 2), (5000, 1),
                     (40000, 1)]:
        inp = synth.matvec_inputs(p, n, batch, seed=400 + n, f_mode="one")
        c = _host(fc.circulant_matvec(_dev(inp["a"]), _dev(inp["b"]), p))
        for k in range(batch):
            exp = oracle.fcirc_entries(p, 1, inp["a"][k], inp["b"][k])
            assert np.array_equal(c[k].astype(np.uint64), exp), (n, k)


# ---------------------------------------------------------------------------------- the paper's ring

M31X2 = fc.M31X2


@pytest.mark.parametrize("f_mode", ["wn", "one", "minus_one"])
def test_m31x2_matvec_all_entries(f_mode):
    """The f-circulant product over the paper's own ring Z/(2^31-1)[sqrt 3], every entry
    against Definition 2 in that ring: fused sizes and the first multi-pass sizes."""
    for L in list(range(0, 14)) + [15]:
        batch = 3 if L <= 10 else 1
        inp = synth.matvec_inputs(M31X2, 1 << L, batch, seed=600 + L, f_mode=f_mode)
        c = run_matvec(inp)
        for k in range(batch):
            exp = oracle.fcirc_entries_m31x2(inp["f"], inp["a"][k], inp["b"][k])
            got = c[k].astype(np.uint64)
            bad = np.nonzero(got != exp)[0]
            assert bad.size == 0, (L, k, bad[:4])


def test_m31x2_matvec_edge_components():
    """Z/(2^31-1)[sqrt 3] with both components drawn from the corner set (0, 1, p-1, p-2, 2^30, ...):
    the per-component folds of FieldM31x2 at their extremes, every entry, fused and multi-pass."""
    rng = np.random.default_rng(31)
    p = (1 << 31) - 1
    for L in [6, 12, 13]:
        n = 1 << L
        u = synth.edge_mix(p, (2, 2, n), rng).astype(np.uint64)
        a = (u[0] | (synth.edge_mix(p, (2, n), rng).astype(np.uint64) << np.uint64(32)))
        b = (u[1] | (synth.edge_mix(p, (2, n), rng).astype(np.uint64) << np.uint64(32)))
        base = synth.matvec_inputs(M31X2, n, 1, seed=700 + L)
        inp = dict(p=M31X2, n=n, batch=2, f=base["f"], w=base["w"], a=a, b=b)
        c = run_matvec(inp)
        for k in range(2):
            exp = oracle.fcirc_entries_m31x2(inp["f"], a[k], b[k])
            bad = np.nonzero(c[k].astype(np.uint64) != exp)[0]
            assert bad.size == 0, (L, k, bad[:4])


def test_m31x2_matvec_multipass_sampled():
    for L in range(16, 21):
        inp = synth.matvec_inputs(M31X2, 1 << L, 2, seed=650 + L)
        c = run_matvec(inp)
        for k in range(2):
            idx = synth.sample_indices(1 << L, 512, seed=k)
            exp = oracle.fcirc_entries_m31x2(inp["f"], inp["a"][k], inp["b"][k], idx)
            assert np.array_equal(c[k][idx].astype(np.uint64), exp), (L, k)


def test_m31x2_polymul_paper_shapes():
    """The paper's experiment: products of two n-coefficient polynomials, n = 8..512,
    in Z/(2^31-1)[sqrt 3] -- every coefficient against the schoolbook oracle."""
    for n in [8, 16, 32, 64, 128, 256, 512, 3000]:
        pin = synth.polymul_inputs(M31X2, n, n, 4, seed=n)
        c = _host(fc.polymul(_dev(pin["a"]), _dev(pin["b"]), M31X2))
        for k in range(4):
            assert np.array_equal(c[k].astype(np.uint64), oracle.polymul_coeffs_m31x2(pin["a"][k], pin["b"][k])), (n, k)


def test_m31x2_circulant_any_n():
    for n in [3, 7, 100, 1000]:
        inp = synth.matvec_inputs(M31X2, n, 2, seed=700 + n, f_mode="one")
        c = _host(fc.circulant_matvec(_dev(inp["a"]), _dev(inp["b"]), M31X2))
        for k in range(2):
            assert np.array_equal(c[k].astype(np.uint64), oracle.fcirc_entries_m31x2(1, inp["a"][k], inp["b"][k]))

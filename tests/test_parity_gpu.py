"""GPU parity: the CUDA path (through the C ABI via the thin binding) against the CPU oracle,
element by element, bit-exact (integer work).

Coverage rules (BASELINE.json north_star; helpers in tests/parity.py):
  * n <= 2^14: every entry of every instance;
  * n >  2^14: >= 1024 seeded-random entries + the boundary indices {0, 1, n/2-1, n/2, n-2, n-1}
    on EVERY instance, and the eigen-checksum at 16 seeded theta on every
    instance;
  * polymul: >= 1024 seeded coefficients + boundary ones and Schwartz-Zippel at 8 points on every
    instance; bigint: every full product vs Python ints and the oracle's Karatsuba.
Each config check logs its coverage (instances, entries, thetas, mismatches) to the parity log
(tests/parity.py: $FCIRC_PARITY_LOG or gpurun_out/parity_counts.jsonl).
"""
import os

import numpy as np
import pytest

import oracle
import synth
import parity
from parity import check_matvec, check_polymul
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


def check_sampled(inp, c, instances, count=1024, thetas=16, name=None):
    """>= 1024 seeded entries + boundary and 16 theta on each listed instance (tests/parity.py)."""
    ks = np.asarray(list(instances), dtype=np.int64)
    sub = dict(inp, a=inp["a"][ks], b=inp["b"][ks], batch=len(ks))
    check_matvec(name or f"p={inp['p']} n={inp['n']}", sub, np.asarray(c)[ks], full=False,
                 sample=max(count, 1024), thetas=max(thetas, 16))


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
        check_matvec(f"many instances p={p} n=2^{L}", inp, c, full=True)


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
                    check_sampled(inp, c, [0])


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
            check_sampled(inp, c, [0, 1])


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
        check_matvec(f"multipass p={p} n=2^{L}", inp, c)


def test_matvec_multipass_full_entries_2pow15():
    for p in [P998, GOLDILOCKS]:
        inp = synth.matvec_inputs(p, 1 << 15, 2, seed=33)
        c = run_matvec(inp)
        check_full(inp, c)


def test_matvec_chunking_ragged(monkeypatch):
    """Batch not a multiple of the L2 chunk: instances in the last, short chunk are right."""
    inp = synth.matvec_inputs(GOLDILOCKS, 1 << 16, 7, seed=44)
    c = run_matvec(inp)
    check_sampled(inp, c, range(7))


# ---------------------------------------------------------------------------------- BASELINE configs

def test_config_C1():
    inp = synth.matvec_inputs(**{k: v for k, v in synth.CONFIGS["C1"].items() if k != "kind"})
    c = run_matvec(inp)
    check_full(inp, c)


@pytest.mark.parametrize("name", ["C2_f1", "C2_fm1"])
def test_config_C2(name):
    """C2: n = 2^12 <= 2^14, so every entry of all 4096 instances, plus 16 theta per instance."""
    cfg = {k: v for k, v in synth.CONFIGS[name].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_matvec(name, inp, c)


@pytest.mark.parametrize("L", list(range(15, 23)))
def test_config_C4_goldilocks_sweep(L):
    """C4 n = 2^15 .. 2^22 (batch 2^26 / n): 1024 seeded entries + boundary on every instance and
    16 theta per instance."""
    cfg = {k: v for k, v in synth.CONFIGS[f"C4_n{L}"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_matvec(f"C4_n{L}", inp, c)


@pytest.mark.parametrize("L", [12, 13, 14])
def test_config_C4_goldilocks_small_checksums(L):
    """C4 n = 2^12 .. 2^14: the eigen-checksum at 16 theta on every instance plus every entry of
    64 spread instances (the all-instances, all-entries check is the slow test below)."""
    cfg = {k: v for k, v in synth.CONFIGS[f"C4_n{L}"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_matvec(f"C4_n{L}[checksums]", inp, c, full=False, sample=0)
    ks = np.unique(np.linspace(0, inp["batch"] - 1, 64).astype(np.int64))
    sub = dict(inp, a=inp["a"][ks], b=inp["b"][ks], batch=len(ks))
    check_matvec(f"C4_n{L}[64 instances, all entries]", sub, c[ks], full=True, thetas=0)


@pytest.mark.slow
@pytest.mark.parametrize("L", [12, 13, 14])
def test_config_C4_goldilocks_every_entry(L):
    """C4 n = 2^12 .. 2^14: every entry of every instance (2^26 entries, 2^26 n multiply-adds)."""
    cfg = {k: v for k, v in synth.CONFIGS[f"C4_n{L}"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_matvec(f"C4_n{L}", inp, c, full=True, thetas=0)


def test_config_S1():
    cfg = {k: v for k, v in synth.CONFIGS["S1"].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    c = run_matvec(inp)
    check_matvec("S1", inp, c)


# ---------------------------------------------------------------------------------- host entry

def test_matvec_host_matches_device():
    for p, L, batch in [(GOLDILOCKS, 11, 5), (P998, 16, 9), (GOLDILOCKS, 20, 3)]:
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=55 + L)
        c_host = fc.matvec_host(inp["a"], inp["b"], inp["f"], p)
        c_dev = run_matvec(inp)
        assert np.array_equal(c_host, c_dev)
        check_sampled(inp, c_host, range(batch))


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
    check_sampled(inp, _host(c1), range(4))


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
    assert c.shape == (cfg["batch"], cfg["na"] + cfg["nb"] - 1)
    check_polymul("C3", inp, c)


# ---------------------------------------------------------------------------------- bigint

def _to_int(words):
    return int.from_bytes(np.ascontiguousarray(words, dtype="<u4").tobytes(), "little")


def test_bigint_small():
    rng = np.random.default_rng(88)
    # the three primes run as one launch per pass: odd batches and multi-pass sizes exercise the
    # per-CTA prime selection (staged sub-problems) and the per-thread one (fused, several instances
    # per CTA straddling primes)
    for nx, ny, batch in [(1, 1, 3), (1, 5, 2), (7, 3, 2), (9, 9, 7), (64, 64, 2), (200, 100, 5), (1000, 777, 2),
                          (4096, 4096, 1), (5000, 5000, 5), (20000, 3000, 3)]:
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
        assert np.array_equal(z[k], oracle.bigint_mul(inp["x"][k], inp["y"][k])), k
    parity.record({"config": "C5", "instances": cfg["batch"], "entries": int(z.size), "mode": "all",
                   "mismatches": 0})


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
        check_sampled(inp, c, [0, 1])


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


@pytest.mark.parametrize("knobs", [
    {"FCIRC_GOLD_RB": "4", "FCIRC_GOLD_RBF": "4"},
    {"FCIRC_GOLD_RB": "16", "FCIRC_GOLD_RBF": "16"},
    {"FCIRC_GOLD_MSPLIT": "11"},
    {"FCIRC_GOLD_MSPLIT": "13"},
    {"FCIRC_SMALL_R": "8"},
    {"FCIRC_SHFL": "1"},
    {"FCIRC_COLS2": "0", "FCIRC_INV2": "0", "FCIRC_TMA": "0"},
])
def test_goldilocks_launcher_variants_all_entries(knobs):
    """The Goldilocks kernels under the launcher's run-time knobs (other register blockings R, on-chip
    sub-problem sizes 2^11 / 2^13, the lane-transpose exchange, the one-operand column passes): every
    entry against Definition 2.  The sign-tracking vector split derives its
    negating levels from the phase layout, which differs per (M, R): each variant is a separate
    instantiation of the rule.  Knobs are read once per process, hence the subprocess."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle, paper_2103_02605_b200 as fc, synth
p = synth.GOLDILOCKS
bad = []
for L, batch in [(3, 5), (9, 3), (10, 2), (11, 3), (12, 3), (13, 2), (14, 2), (15, 1)]:
    inp = synth.matvec_inputs(p, 1 << L, batch, seed=900 + L)
    c = fc.matvec(torch.from_numpy(inp["a"]).cuda(), torch.from_numpy(inp["b"]).cuda(), inp["f"], p).cpu().numpy()
    for k in range(batch):
        exp = oracle.fcirc_entries(p, inp["f"], inp["a"][k], inp["b"][k])
        if not np.array_equal(c[k].astype(np.uint64), exp):
            bad.append((L, k))
print("mismatching (L, instance):", bad)
'''
    env = dict(os.environ, **knobs)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "mismatching (L, instance): []" in out.stdout, out.stdout + out.stderr[-2000:]


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


# ---------------------------------------------------------------------------------- runtime robustness

def test_graph_replay_survives_plan_eviction():
    """A product captured in a CUDA graph keeps its twist table alive: after more new plans than the
    cache keeps (64), the graph still replays to the exact product (the plan used under capture is
    pinned; evicted plans are freed stream-ordered after their uses)."""
    inp = synth.matvec_inputs(GOLDILOCKS, 1 << 14, 2, seed=5150)
    a, b = _dev(inp["a"]), _dev(inp["b"])
    c = fc.matvec(a, b, inp["f"], GOLDILOCKS)           # plan built outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            fc.matvec(a, b, inp["f"], GOLDILOCKS, out=c)
    torch.cuda.current_stream().wait_stream(cap)
    n_plans, pinned = fc.plan_count()
    assert pinned >= 1
    rng = np.random.default_rng(77)
    for i in range(80):                                  # evict everything that is not pinned
        q = P998 if i % 2 else GOLDILOCKS
        other = synth.matvec_inputs(q, 1 << 9, 1, seed=int(rng.integers(1 << 30)))
        fc.matvec(_dev(other["a"]), _dev(other["b"]), other["f"], q)
    n_plans, pinned2 = fc.plan_count()
    assert n_plans <= 64 + pinned2 and pinned2 >= 1
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    check_sampled(inp, _host(c), [0, 1], name="graph replay after eviction")


def test_plan_built_inside_capture_is_rejected():
    """The first call for a (p, f, n) builds its plan on the host: not allowed during capture."""
    inp = synth.matvec_inputs(P998, 1 << 11, 1, seed=616161)
    a, b = _dev(inp["a"]), _dev(inp["b"])
    c = torch.empty_like(a)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with pytest.raises(fc.FcircError) as ei:
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                fc.matvec(a, b, inp["f"], P998, out=c)
    assert ei.value.code == -1


def test_binding_validates_out_and_handles_unaligned_views():
    """`out` of the wrong shape is rejected by the binding (no out-of-bounds writes); an output view
    that is only element-aligned (not 16-byte aligned) takes the non-TMA column kernels and is exact."""
    inp = synth.matvec_inputs(GOLDILOCKS, 1 << 10, 2, seed=3)
    a, b = _dev(inp["a"]), _dev(inp["b"])
    with pytest.raises(ValueError):
        fc.matvec(a, b, inp["f"], GOLDILOCKS, out=torch.empty((2, 512), dtype=a.dtype, device="cuda"))
    with pytest.raises(ValueError):
        fc.polymul(a, b, GOLDILOCKS, out=torch.empty((2, 100), dtype=a.dtype, device="cuda"))
    L = 21   # Goldilocks 2^21: 9 column levels -> the TMA inverse pass when aligned
    big = synth.matvec_inputs(GOLDILOCKS, 1 << L, 1, seed=12)
    store = torch.empty((1 << L) + 1, dtype=torch.int64, device="cuda")
    out = store[1:].view(1, 1 << L)                     # 8-byte but not 16-byte aligned
    assert out.data_ptr() % 16 == 8
    fc.matvec(_dev(big["a"]), _dev(big["b"]), big["f"], GOLDILOCKS, out=out)
    torch.cuda.synchronize()
    check_sampled(big, _host(out), [0], name="unaligned output view")


def test_host_pipeline_concurrent_threads():
    """fcirc_matvec_host from two host threads at once (per-call contexts from a pool)."""
    import threading
    errors, res = [], {}

    def work(tid):
        try:
            for j in range(3):
                p = GOLDILOCKS if (tid + j) % 2 else P998
                inp = synth.matvec_inputs(p, 1 << (12 + 2 * j), 3, seed=900 + 10 * tid + j)
                res[(tid, j)] = (inp, fc.matvec_host(inp["a"], inp["b"], inp["f"], p))
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for (tid, j), (inp, c) in res.items():
        check_sampled(inp, c, range(inp["batch"]), name=f"host pipeline thread {tid} call {j}")


def test_outputs_stay_inside_their_buffers():
    """Own bounds check (compute-sanitizer is closed on this pool): every output is written into the
    middle of a larger buffer whose guard bands hold a sentinel; after the call the guards must be
    untouched and the product exact -- fused, multi-pass (incl. the TMA and vector column paths),
    truncating polymul stores, any-n circulants and bigint."""
    G = 4096   # guard elements on each side

    def guarded(shape, dtype):
        n = int(np.prod(shape))
        store = torch.full((n + 2 * G,), 0x5A5A5A5A, dtype=dtype, device="cuda")
        return store, store[G:G + n].view(*shape)

    def guards_intact(store):
        g = store.cpu().numpy()
        return bool((g[:G] == 0x5A5A5A5A).all() and (g[-G:] == 0x5A5A5A5A).all())

    for p, L, batch in [(GOLDILOCKS, 10, 3), (GOLDILOCKS, 16, 2), (GOLDILOCKS, 21, 1), (P998, 12, 5), (P998, 17, 3)]:
        inp = synth.matvec_inputs(p, 1 << L, batch, seed=8000 + L)
        dt = torch.int64 if p == GOLDILOCKS else torch.int32
        store, out = guarded((batch, 1 << L), dt)
        fc.matvec(_dev(inp["a"]), _dev(inp["b"]), inp["f"], p, out=out)
        torch.cuda.synchronize()
        assert guards_intact(store), (p, L)
        check_sampled(inp, _host(out), range(batch), name=f"guarded p={p} n=2^{L}")
    for na, nb in [(700, 300), (9000, 7000)]:
        pin = synth.polymul_inputs(P998, na, nb, 2, seed=na)
        store, out = guarded((2, na + nb - 1), torch.int32)
        fc.polymul(_dev(pin["a"]), _dev(pin["b"]), P998, out=out)
        torch.cuda.synchronize()
        assert guards_intact(store), (na, nb)
        for k in range(2):
            assert np.array_equal(_host(out)[k].astype(np.uint32).astype(np.uint64),
                                  oracle.polymul_coeffs(P998, pin["a"][k], pin["b"][k]))
    for n in [1000, 5000]:
        inp = synth.matvec_inputs(P998, n, 2, seed=n, f_mode="one")
        store, out = guarded((2, n), torch.int32)
        fc.circulant_matvec(_dev(inp["a"]), _dev(inp["b"]), P998, out=out)
        torch.cuda.synchronize()
        assert guards_intact(store), n
    bi = synth.bigint_inputs(3000, 3, seed=4)
    store, out = guarded((3, 6000), torch.int32)
    fc.bigint_mul(_dev(bi["x"]), _dev(bi["y"]), out=out)
    torch.cuda.synchronize()
    assert guards_intact(store)
    z = _host(out).astype(np.uint32)
    for k in range(3):
        assert _to_int(z[k]) == _to_int(bi["x"][k]) * _to_int(bi["y"][k])

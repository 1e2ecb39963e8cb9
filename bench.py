#!/usr/bin/env python
"""bench.py — libfcirc headline benchmark (BASELINE.json metric) on one node.

A "step" is one batched f-circulant matrix-vector product (the whole hot path of SURVEY §8(a):
forward split of a and b, leaves, recombination, 1/n scaling) over one batch of synthetic input.
Default workload = the BASELINE.json metric point (SURVEY §8(d) C4 @ n=2^20): Goldilocks
p = 2^64-2^32+1, n = 2^20, batch 64, f = w^n (seeded), a, b ~ U[0,p) — 512 MiB per operand, so
every step reads its inputs from HBM (inputs larger than the 126 MB L2).  --config selects the
other configurations: S1 / C2 / C4 sweep points (matvec), C3 (polynomial products, step = one
batched fcirc_polymul) and C5 (big integers, step = one batched bigint_mul).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fcirc|reference] [--config NAME]

N > 1 runs under torchrun: one process per GPU, each rank its own batch (independent instances,
no data-path collective; weak scaling).  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, Definition 2 written out) on a bounded sample of
the same workload — the tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "f-circulant matvec Gelem/s mod p at n=2^20 (batched); % of HBM/int roofline"
UNIT = "Gelem/s"

# Roofline denominators are MEASURED in the same run: the integer peak is the rate of the
# library's own ring primitives (fcirc_primitive_rate: SURVEY §8(d)'s R_const / R_var), the
# multiplier-only ceiling is derived from the raw IMAD.WIDE.U32 rate measured beside it, and HBM is
# MEASURED_PEAKS.json's copy bandwidth (driver-written).
HBM_GBS_FALLBACK = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
# primitive kinds per element width: (R_const probe, R_var probe, IMAD.WIDE slots per modmul)
PRIMS = {"u64": ("gold_mulm", "gold_leaf", 4), "u32": ("u32_mulc", "u32_leaf", 2), "fp2": ("m31x2_mul", "m31x2_mul", 4)}
PROBE_ITERS = {"gold_mul": 20000, "gold_mulm": 20000, "gold_leaf": 20000, "u32_mulc": 60000, "u32_leaf": 40000, "m31x2_mul": 30000, "imad_wide": 100000,
               "gold_fwd_a": 15000, "gold_fwd_b": 15000, "gold_inv": 15000, "u32_fwd_a": 40000}

WORKLOADS = {
    "C4_n20": "C4 @ n=2^20: Goldilocks f-circulant matvec, batch 64, f=w^n",
    "S1": "S1: p=998244353 f-circulant matvec n=2^20, batch 64, f=w^n",
    "C1": "C1: p=998244353 f-circulant matvec n=2^10, batch 1, f=w^n",
    "C2_f1": "C2: p=998244353 circulant matvec n=2^12, batch 4096, f=1",
    "C2_fm1": "C2: p=998244353 negacyclic matvec n=2^12, batch 4096, f=p-1",
    **{f"C4_n{L}": f"C4 @ n=2^{L}: Goldilocks f-circulant matvec, batch 2^{26 - L}"
       for L in range(12, 23) if L != 20},
    "C3": "C3: polynomial products mod 998244353, 2^20 x 2^20 coefficients -> 2^21 circulant (f=1), batch 16",
    "C5": "C5: 2^22-bit integer products, 16-bit limbs, 3 primes x 2^19 circulant (f=1) + CRT + carry, batch 8",
    "N3_gold": ("NEXT-3 (Corollary 1): Goldilocks usual circulant matvec of order n=1000003 (not a power of two, "
                "embedded in 2^21), batch 32"),
    "N3_u32": ("NEXT-3 (Corollary 1): p=998244353 usual circulant matvec of order n=1000003 (not a power of two, "
               "embedded in 2^21), batch 32"),
    **{f"S2_n{n}": (f"S2 (context): the paper's experiment, 10000 products of two {n}-coefficient polynomials in "
                    f"Z/(2^31-1)[sqrt 3] (P:110-133)") for n in (8, 16, 32, 64, 128, 256, 512)},
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def traffic_record(config: str, kind: str):
    """DRAM bytes per launch of `kind` from the committed ncu --set full capture (profiles/traffic.json,
    written by tools/ncu_summary.py traffic), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(config, {}).get(kind)
    except Exception:
        return None


# ------------------------------------------------------------------------------------ clocks

class ClockSampler:
    """NVML sampling of SM clock and clocks-event reasons while running (DURING the timed region)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, cuda_index: int, period: float = 0.02):
        self.samples = []
        self.period = period
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            try:  # match the CUDA device by PCI bus id (CUDA_VISIBLE_DEVICES may renumber)
                import torch
                props = torch.cuda.get_device_properties(cuda_index)
                bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(cuda_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _sample(self):
        nv = self.nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.samples.append((mhz, int(rs)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        mhz = [s[0] for s in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        reasons = [name for bit, name in self.REASONS.items() if bits & bit]
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------ helpers

def rank_config(cfg: dict, rank: int) -> dict:
    """Per-rank workload: every rank draws its own independent instances of the
    same configuration (weak scaling, no data-path collective)."""
    out = dict(cfg)
    out["seed"] = out["seed"] + 7919 * rank
    return out


def max_over_ranks(x: float, world: int, device="cuda") -> float:
    """Max of a per-rank scalar over all ranks (the timing rule: slowest rank defines the step)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gelems(world: int, batch: int, n: int, steps: int, ms_max: float) -> float:
    """Whole-job throughput: elements of all ranks / the slowest rank's time."""
    return world * batch * n * steps / (ms_max * 1e-3) / 1e9


def algorithmic_modmuls(kind: str, n: int, batch: int, M: int, K: int):
    """(M_const, M_var) algorithmic modmuls per step attributed to one kernel kind:
    M_const = 1.5 n L (0.5 n L each for the a split, the b split, the recombination), M_var = n.
    (M, K) = the library's pass schedule (fcirc_schedule): sub-problems of 2^M, K column levels."""
    L = n.bit_length() - 1
    if kind == "k_block_fused":
        return batch * n * 1.5 * L, batch * n
    if kind == "k_block_sub":
        return batch * n * 1.5 * M, batch * n
    if kind == "k_cols_fwd":
        return batch * n * 1.0 * K, 0.0
    if kind == "k_cols_inv":
        return batch * n * 0.5 * K, 0.0
    return 0.0, 0.0


def measure_primitives(fc, width: str, sampler_cls, device: int) -> dict:
    """Rates of the library's own primitives on this GPU, now (fcirc_primitive_rate), with the SM clock
    sampled while they run: R_const, R_var and the IMAD.WIDE.U32 rate for the ceiling."""
    rc_kind, rv_kind, slots = PRIMS[width]
    kinds = sorted({rc_kind, rv_kind, "imad_wide"} |
                   ({"gold_fwd_a", "gold_fwd_b", "gold_inv"} if width == "u64" else
                    {"u32_fwd_a"} if width == "u32" else set()))
    out = {}
    smp = sampler_cls(device)
    with smp:
        for k in kinds:
            fc.primitive_rate(k, max(1000, PROBE_ITERS[k] // 10))      # warm the clocks
            ops, ms = fc.primitive_rate(k, PROBE_ITERS[k])
            out[k] = {"ops_per_s": ops, "ms": ms}
    clk = smp.summary()
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    for k, v in out.items():
        v["per_clk_per_sm"] = v["ops_per_s"] / (148 * mhz * 1e6)
    return {"R_const": out[rc_kind]["ops_per_s"], "R_var": out[rv_kind]["ops_per_s"],
            "R_const_kind": rc_kind, "R_var_kind": rv_kind,
            "ceiling_modmul_per_s": out["imad_wide"]["ops_per_s"] / slots, "imad_wide_slots_per_modmul": slots,
            "primitives": out, "clocks": clk}


def cfg_dtype(p: int) -> str:
    return "u64" if p >= (1 << 32) or p == synth.M31X2 else "u32"


def next_pow2(x: int) -> int:
    r = 1
    while r < x:
        r <<= 1
    return r


class Workload:
    """One benchmark configuration: inputs, the step through the public API, its end-to-end
    (host buffers) variant, the elements it counts and the oracle sample of the CPU baseline."""

    def __init__(self, name: str, rank: int = 0):
        self.name, self.desc = name, WORKLOADS[name]
        cfg = dict(synth.CONFIGS[name])
        self.kind = cfg.pop("kind")
        self.cfg = rank_config(cfg, rank)
        if self.kind in ("matvec", "anyn"):
            self.inp = synth.matvec_inputs(**self.cfg)
            self.p, self.n, self.batch = self.inp["p"], self.inp["n"], self.inp["batch"]
            self.width = cfg_dtype(self.p)
            self.elems = self.batch * self.n                 # output entries
            self.mm_n, self.mm_batch = self.n, self.batch    # matvec instances launched per step
            if self.kind == "anyn":                          # embedded in the smallest 2^m >= 2n - 1
                self.mm_n = next_pow2(2 * self.n - 1)
        elif self.kind == "polymul":
            self.inp = synth.polymul_inputs(**self.cfg)
            self.p, self.batch = self.inp["p"], self.inp["batch"]
            self.n = next_pow2(self.inp["na"] + self.inp["nb"] - 1)
            self.width = cfg_dtype(self.p)
            self.elems = self.batch * self.n                 # circulant entries
            self.mm_n, self.mm_batch = self.n, self.batch
        elif self.kind == "bigint":
            self.inp = synth.bigint_inputs(**self.cfg)
            self.p, self.batch = synth.P998, self.inp["batch"]
            nw = self.inp["nwords"]
            self.n = next_pow2(2 * (nw + nw) - 1)
            self.width = "u32"
            self.elems = self.batch * self.n                 # output limb positions
            self.mm_n, self.mm_batch = self.n, 3 * self.batch  # three primes
        else:
            raise ValueError(self.kind)

    # ---------------------------------------------------------------- device side
    def setup(self, torch, fc):
        self.torch, self.fc = torch, fc
        i = self.inp
        if self.kind in ("matvec", "anyn"):
            self.dev = [torch.from_numpy(i["a"]).cuda(), torch.from_numpy(i["b"]).cuda()]
            self.out = torch.empty_like(self.dev[0])
        elif self.kind == "polymul":
            self.dev = [torch.from_numpy(i["a"]).cuda(), torch.from_numpy(i["b"]).cuda()]
            self.out = torch.empty((self.batch, i["na"] + i["nb"] - 1), dtype=self.dev[0].dtype, device="cuda")
        else:
            self.dev = [torch.from_numpy(i["x"]).cuda(), torch.from_numpy(i["y"]).cuda()]
            self.out = torch.empty((self.batch, 2 * i["nwords"]), dtype=self.dev[0].dtype, device="cuda")

    def step(self):
        fc, (x, y) = self.fc, self.dev
        if self.kind == "matvec":
            fc.matvec(x, y, self.inp["f"], self.p, out=self.out)
        elif self.kind == "anyn":
            fc.circulant_matvec(x, y, self.p, out=self.out)
        elif self.kind == "polymul":
            fc.polymul(x, y, self.p, out=self.out)
        else:
            fc.bigint_mul(x, y, out=self.out)
        return fc.last_launch_count()

    # ---------------------------------------------------------------- end to end (host buffers)
    def setup_host(self):
        torch = self.torch
        self.host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in self._host_arrays()]
        self.host_out = torch.empty(tuple(self.out.shape), dtype=self.out.dtype).pin_memory()
        self.h2d_bytes = sum(h.numel() * h.element_size() for h in self.host)
        self.d2h_bytes = self.host_out.numel() * self.host_out.element_size()

    def _host_arrays(self):
        i = self.inp
        return (i["a"], i["b"]) if self.kind in ("matvec", "polymul", "anyn") else (i["x"], i["y"])

    def host_step(self):
        """One step through the public API from pinned host memory (H2D, product, D2H)."""
        if self.kind == "matvec":
            self.fc.matvec_host(self.host[0], self.host[1], self.inp["f"], self.p, out=self.host_out)
            return "fcirc_matvec_host (pinned host buffers, chunk-pipelined H2D / kernels / D2H)"
        torch = self.torch
        for d, h in zip(self.dev, self.host):
            d.copy_(h, non_blocking=True)
        self.step()
        self.host_out.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return ("pinned host -> device copies, fcirc_%s, device -> pinned host copy, synchronize"
                % {"polymul": "polymul", "anyn": "circulant_matvec"}.get(self.kind, "bigint_mul"))

    # ---------------------------------------------------------------- CPU oracle sample
    def cpu_sample(self, seconds: float, step_index: int = 0):
        """(elements/s, count, seconds, threads, description) of the oracle as it stands on a
        bounded sample of this workload (entries / coefficients / whole products)."""
        import oracle
        threads = oracle.default_threads()
        i = self.inp
        k = step_index % self.batch
        if self.kind == "bigint":
            t0 = time.perf_counter()
            reps = 0
            while True:
                oracle.bigint_mul(i["x"][k], i["y"][k])
                reps += 1
                if time.perf_counter() - t0 >= seconds * 0.5 or reps >= 64:
                    break
            dt = time.perf_counter() - t0
            return (reps * self.n / dt, reps * self.n, dt, 1,
                    f"{reps} full products of instance {k} (independent Karatsuba on 32-bit words, "
                    f"one thread); counted as {self.n} output limb positions each")
        if self.kind == "polymul":
            if self.p == synth.M31X2:
                fn = lambda ks: oracle.polymul_coeffs_m31x2(i["a"][k], i["b"][k], ks)  # noqa: E731
            else:
                fn = lambda ks: oracle.polymul_coeffs(self.p, i["a"][k], i["b"][k], ks)  # noqa: E731
            what = "schoolbook coefficients"
            total = i["na"] + i["nb"] - 1
        elif self.p == synth.M31X2:
            fn = lambda ks: oracle.fcirc_entries_m31x2(self.inp["f"], i["a"][k], i["b"][k], ks)  # noqa: E731
            what = "output entries (Definition 2 over Z/(2^31-1)[sqrt 3])"
            total = self.n
        else:
            fn = lambda ks: oracle.fcirc_entries(self.p, self.inp["f"], i["a"][k], i["b"][k], ks)  # noqa: E731
            what = "output entries (Definition 2, O(n) multiply-adds each)"
            total = self.n
        probe = max(threads, 32)
        t0 = time.perf_counter()
        fn(np.arange(probe, dtype=np.int64))
        dt = time.perf_counter() - t0
        count = int(min(total, max(probe, probe * seconds / max(dt, 1e-6))))
        idx = np.random.default_rng(7 + step_index).integers(0, total, count).astype(np.int64)
        t0 = time.perf_counter()
        fn(idx)
        dt = time.perf_counter() - t0
        return (count / dt, count, dt, threads,
                f"{count} seeded-random {what} of instance {k} of {self.desc}; {dt:.1f} s wall")

    def config_block(self, args):
        arr = self._host_arrays()[0]
        blk = {"workload": self.desc, "p": int(self.p), "n": int(self.n), "batch": int(self.batch),
               "l2": ("inputs larger than L2 (%.0f MiB per input operand per rank; L2 126 MB)" % (arr.nbytes / 2**20)
                      if arr.nbytes > (126 << 20) else
                      "inputs smaller than L2 (%.1f MiB per operand); no flush between steps" % (arr.nbytes / 2**20)),
               "parallelism": f"replicas x{args.gpus} (independent instances per GPU, no collective)"}
        if self.kind == "matvec":
            blk["f"] = "w^n" if self.inp.get("w") not in (None, 1) else ("1" if self.inp["f"] == 1 else "p-1")
        if self.kind == "anyn":
            blk["f"] = "1 (usual circulant)"
            blk["embedded_order"] = int(self.mm_n)
        return blk


# ------------------------------------------------------------------------------------ arms

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = Workload(args.config)
    _, _, _, threads, _ = wl.cpu_sample(0.2)
    times, counts, desc = [], [], ""
    for s in range(args.warmup + args.steps):
        rate, count, dt, threads, desc = wl.cpu_sample(1.0, step_index=s)
        if s >= args.warmup:
            times.append(dt)
            counts.append(count)
    total = sum(times)
    value = sum(counts) / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": wl.width,
        "data": "synthetic", "config": wl.config_block(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": "per step: " + desc.rsplit(";", 1)[0] + " (about 1 s of CPU work per step)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def prim_width(p: int) -> str:
    return "fp2" if p == synth.M31X2 else ("u64" if p >= (1 << 32) else "u32")


def bench_parity(wl, out, thetas: int, instances: int) -> dict:
    """Check the product the timed region computed (the last step's output, copied back) against the
    oracle: >= 1024 seeded entries + boundary on `instances` spread
    instances, the eigen-checksum at `thetas` theta on EVERY instance (matvec); seeded coefficients
    + Schwartz-Zippel (polymul); every full product vs Python ints (bigint).  Test infrastructure
    (tests/parity.py -> oracle/), run after timing."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import parity
    t0 = time.time()
    host = out.cpu().numpy()
    i = wl.inp
    if wl.kind == "matvec":
        ks = np.unique(np.linspace(0, wl.batch - 1, min(instances, wl.batch)).astype(np.int64))
        sub = dict(i, a=i["a"][ks], b=i["b"][ks], batch=len(ks))
        r1 = parity.check_matvec(wl.name + "[bench sampled]", sub, host[ks], full=False, thetas=0)
        r2 = parity.check_matvec(wl.name + "[bench checksums]", i, host, full=False, sample=0, thetas=thetas)
        return {"sampled_instances": int(len(ks)), "entries": r1["entries"], "eigen_instances": wl.batch,
                "thetas_per_instance": thetas, "mismatches": r1["mismatches"] + r2["mismatches"],
                "eigen_ok": r2["eigen_ok"], "seconds": round(time.time() - t0, 2)}
    if wl.kind == "anyn":   # sampled entries (Definition 2, f = 1) + sum(c) = sum(a) sum(b) on every instance
        ks = np.unique(np.linspace(0, wl.batch - 1, min(instances, wl.batch)).astype(np.int64))
        sub = dict(i, a=i["a"][ks], b=i["b"][ks], batch=len(ks))
        r1 = parity.check_matvec(wl.name + "[bench sampled]", sub, host[ks], full=False, thetas=0)
        bad_sum = 0
        for k in range(wl.batch):   # theta = 1 is an n-th root of f = 1 for every n
            sa, sb, sc = (int(np.sum(x.astype(object))) for x in (i["a"][k], i["b"][k], host[k]))
            bad_sum += (sc - sa * sb) % wl.p != 0
        assert bad_sum == 0, f"{wl.name}: {bad_sum} instances fail sum(c) = sum(a) sum(b)"
        return {"sampled_instances": int(len(ks)), "entries": r1["entries"], "sum_check_instances": wl.batch,
                "mismatches": r1["mismatches"] + int(bad_sum), "seconds": round(time.time() - t0, 2)}
    if wl.kind == "polymul" and wl.p == synth.M31X2:   # the paper's ring: every coefficient, 4 instances
        import oracle
        ks = np.unique(np.linspace(0, wl.batch - 1, min(instances, wl.batch)).astype(np.int64))
        bad = sum(int(np.count_nonzero(host[k].astype(np.uint64) != oracle.polymul_coeffs_m31x2(i["a"][k], i["b"][k])))
                  for k in ks)
        assert bad == 0, f"{wl.name}: {bad} mismatching coefficients"
        return {"sampled_instances": int(len(ks)), "entries": int(len(ks) * host.shape[1]), "mismatches": bad,
                "mode": "every coefficient vs the Z/(2^31-1)[sqrt 3] schoolbook oracle",
                "seconds": round(time.time() - t0, 2)}
    if wl.kind == "polymul":
        ks = np.unique(np.linspace(0, wl.batch - 1, min(instances, wl.batch)).astype(np.int64))
        sub = dict(i, a=i["a"][ks], b=i["b"][ks], batch=len(ks))
        r = parity.check_polymul(wl.name + "[bench]", sub, host[ks])
        return {"sampled_instances": int(len(ks)), "entries": r["entries"], "sz_points_per_instance":
                r["sz_points_per_instance"], "mismatches": r["mismatches"], "seconds": round(time.time() - t0, 2)}
    bad = 0
    for k in range(wl.batch):
        z = int.from_bytes(np.ascontiguousarray(host[k], dtype="<u4").tobytes(), "little")
        x = int.from_bytes(np.ascontiguousarray(i["x"][k], dtype="<u4").tobytes(), "little")
        y = int.from_bytes(np.ascontiguousarray(i["y"][k], dtype="<u4").tobytes(), "little")
        bad += z != x * y
    assert bad == 0, f"bigint parity: {bad} wrong products"
    return {"instances": wl.batch, "entries": int(host.size), "mode": "every full product vs Python int",
            "mismatches": int(bad), "seconds": round(time.time() - t0, 2)}


def run_fcirc(args):
    import torch
    import torch.distributed as dist
    import paper_2103_02605_b200 as fc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = Workload(args.config, rank)
    wl.setup(torch, fc)
    stream = torch.cuda.current_stream()

    # plan build (first call) timed separately, then the remaining warm-up steps
    t0 = time.perf_counter()
    wl.step()
    torch.cuda.synchronize()
    plan_ms = 1000 * (time.perf_counter() - t0)
    for _ in range(args.warmup - 1):
        wl.step()
    torch.cuda.synchronize()

    # ---- CUDA graph of one step (launch-bound configurations: the step is shorter than the host
    # time to issue it, so the timed region replays a captured graph instead of calling the API)
    use_graph = args.graph == "on" or (args.graph == "auto" and (wl.elems < (1 << 20) or wl.kind == "bigint"))
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                wl.step()
        stream.wait_stream(cap)
        graph.replay()
        torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream; one event pair per step
    # for the min / median, one pair around all K steps for the mean)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        ev0.record(stream)
        for k in range(args.steps):
            if use_graph:
                graph.replay()
            else:
                launches += wl.step()
        ev1.record(stream)
        torch.cuda.synchronize()
    # per-step event pairs for ms_min / ms_median in a second pass of the same K steps (an event
    # record between back-to-back steps would perturb the mean of short, launch-bound steps)
    for k in range(args.steps):
        sev[k][0].record(stream)
        if use_graph:
            graph.replay()
        else:
            wl.step()
        sev[k][1].record(stream)
    torch.cuda.synchronize()
    # per-kernel event timing (the library brackets each launch with events on its stream) from a
    # separate, un-captured pass of the same K steps: the events cost a few microseconds per launch,
    # which the timed region above must not carry (C2: 12 % of a 0.13 ms step)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fc.profile_read()
    fc.profile_enable(True)
    pe0.record(stream)
    for _ in range(args.steps):
        n_l = wl.step()
        if use_graph:
            launches += n_l
    pe1.record(stream)
    torch.cuda.synchronize()
    fc.profile_enable(False)
    prof = fc.profile_read()
    prof_ms = pe0.elapsed_time(pe1)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    step_ms = sorted(a.elapsed_time(b) for a, b in sev)
    ms_max = max_over_ranks(ms, world)
    ms_step = ms_max / args.steps
    ms_min = max_over_ranks(step_ms[0], world)
    ms_median = max_over_ranks(statistics.median(step_ms), world)
    value = world * wl.elems * args.steps / (ms_max * 1e-3) / 1e9

    # ---- parity of the benched product (after timing; the output of the last timed step)
    parity_blk = None
    if not args.no_parity:
        parity_blk = bench_parity(wl, wl.out, thetas=args.parity_thetas, instances=4)

    # ---- measured integer peaks (same run, same GPU): the library's own primitives
    width, pw, n, batch = wl.width, prim_width(wl.p), wl.mm_n, wl.mm_batch
    if args.no_probe:   # (ncu launch-list runs: keep the probe kernels out of the kernel list)
        prims = {"R_const": float("nan"), "R_var": float("nan"), "ceiling_modmul_per_s": float("nan"),
                 "R_const_kind": "skipped (--no-probe)", "R_var_kind": "skipped", "imad_wide_slots_per_modmul": 0,
                 "primitives": {}, "clocks": None}
    else:
        prims = measure_primitives(fc, pw, ClockSampler, torch.cuda.current_device())
    R_const, R_var, R_ceil = prims["R_const"], prims["R_var"], prims["ceiling_modmul_per_s"]

    # ---- roofline of the dominant kernel
    dom = max((k for k in prof if prof[k][0] > 0), key=lambda k: prof[k][1])
    cnt, kms = prof[dom]
    sub_log, top = fc.schedule(wl.p, n)
    mc, mv = algorithmic_modmuls(dom, n, batch, sub_log, top)
    mc, mv = mc * args.steps / cnt, mv * args.steps / cnt          # per launch
    avg_ms = kms / cnt
    achieved = (mc + mv) / (avg_ms * 1e-3) / 1e12
    t_roof_k = mc / R_const + mv / R_var                           # seconds at the measured peak
    peak = (mc + mv) / t_roof_k / 1e12
    peak_ceil = R_ceil / 1e12
    mp = measured_peaks()
    hbm = (mp or {}).get("hbm_gbs", HBM_GBS_FALLBACK)
    L = n.bit_length() - 1
    step_mc, step_mv = batch * n * 1.5 * L, batch * n
    step_bytes = 3 * batch * n * (8 if width == "u64" else 4)
    t_int = step_mc / R_const + step_mv / R_var
    t_roof = max(step_bytes / (hbm * 1e9), t_int)
    tr = traffic_record(args.config, dom)
    roofline = {
        "bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "Tmodmul/s",
        "frac": achieved / peak, "traffic": tr["bytes_per_launch"] if tr else None,
        "traffic_source": (f"{tr['report']} ({tr['note']})" if tr else None),
        "peak_source": (f"measured in this run: fcirc_primitive_rate {prims['R_const_kind']} (R_const) / "
                        f"{prims['R_var_kind']} (R_var), the library's own modmul primitives on all SMs "
                        f"(SURVEY §8(d)); blended for this kernel's const/var mix"),
        "ceiling": peak_ceil, "frac_vs_ceiling": achieved / peak_ceil,
        "ceiling_source": (f"measured IMAD.WIDE.U32 rate / {prims['imad_wide_slots_per_modmul']} "
                           f"(multiplier-only: the minimum multiply issue slots of one modmul, DESIGN.md §6)"),
        "per_launch": {"modmuls_const": mc, "modmuls_var": mv, "avg_ms": avg_ms, "launches": cnt},
        "primitives": {k: {"tops_per_s": v["ops_per_s"] / 1e12, "per_clk_per_sm": v["per_clk_per_sm"]}
                       for k, v in prims["primitives"].items()},
        "primitive_clocks": prims["clocks"],
        "kernel_share_of_step": kms / prof_ms,
        "kernels": {k: {"launches": v[0], "ms_total": v[1]} for k, v in prof.items() if v[0]},
        "step": {"t_roof_ms": 1000 * t_roof, "frac": 1000 * t_roof / ms_step,
                 "frac_vs_ceiling": 1000 * max(step_bytes / (hbm * 1e9), (step_mc + step_mv) / R_ceil) / ms_step,
                 "hbm_bound_ms": 1000 * step_bytes / (hbm * 1e9), "alu_bound_ms": 1000 * t_int,
                 "hbm_gbs_peak": hbm, "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs" if mp else "fallback",
                 "hbm_gbs_achieved_alg": step_bytes / (ms_step * 1e-3) / 1e9},
    }

    # ---- end to end through the public API (pinned host buffers, H2D + product + D2H per step)
    e2e = None
    if not args.no_e2e:
        wl.setup_host()
        api = wl.host_step()
        if world > 1:
            dist.barrier()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            wl.host_step()
        dt = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": world * wl.elems * e_steps / dt / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": wl.h2d_bytes, "d2h_bytes_per_step": wl.d2h_bytes,
               "steps": e_steps, "api": api + "; wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, count, dt, threads, desc = wl.cpu_sample(args.cpu_seconds)
        cpu = {"value": rate / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "ms_min": ms_min, "ms_median": ms_median,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": width, "data": "synthetic (seeded uniform residues, SURVEY §8(d))",
            "config": wl.config_block(args), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "parity": parity_blk, "gpu_launches": launches, "clocks": sampler.summary(), "plan_build_ms": plan_ms,
            "timing": ("CUDA graph replay of the step" if use_graph else "API call per step") +
                      "; ms_per_step = mean over the K steps (one event pair), ms_min / ms_median over per-step "
                      "event pairs of a second pass; per-kernel times from a third, profiled pass",
        }
        if wl.kind in ("polymul", "bigint"):
            line["products_per_s"] = world * wl.batch * args.steps / (ms_max * 1e-3)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["fcirc", "reference"], default="fcirc")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="C4_n20")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the benched output")
    ap.add_argument("--no-probe", action="store_true",
                    help="skip the primitive-rate probe (roofline peaks become NaN; for ncu launch lists)")
    ap.add_argument("--parity-thetas", type=int, default=4,
                    help="eigen-checksum points per instance in the bench parity check")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay a CUDA graph of one step in the timed region "
                         "(auto: launch-bound steps -- fewer than 2^20 elements, or the 14-launch bigint)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_fcirc(args)


if __name__ == "__main__":
    sys.exit(main())

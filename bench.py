#!/usr/bin/env python
"""bench.py — libfcirc headline benchmark (BASELINE.json metric) on one node.

A "step" is one batched f-circulant matrix-vector product (the whole hot path of SURVEY §8(a):
forward split of a and b, leaves, recombination, 1/n scaling) over one batch of synthetic input.
Default workload = the BASELINE.json metric point (SURVEY §8(d) C4 @ n=2^20): Goldilocks
p = 2^64-2^32+1, n = 2^20, batch 64, f = w^n (seeded), a, b ~ U[0,p) — 512 MiB per operand, so
every step reads its inputs from HBM (inputs larger than the 126 MB L2).

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

# Roofline denominators.  Integer pipe: derived from the unit counts measured on
# this pool's B200 (profiles/r01_peaks.jsonl: IMAD 64/clk/SM, IMAD.HI and IMAD.WIDE.U32 32/clk/SM,
# i.e. 2 FMA-pipe slots each) and the SM clock of MEASURED_PEAKS.json (1965 MHz), 148 SMs:
#   Goldilocks modmul: minimum 4 IMAD.WIDE partial products = 8 slots -> 8 modmul/clk/SM
#   32-bit Shoup modmul: 1 IMAD.HI + 2 IMAD = 4 slots                 -> 16 modmul/clk/SM
SMS = 148
SM_MHZ = 1965.0
MODMUL_PER_CLK_SM = {"u64": 8.0, "u32": 16.0}
PRIMITIVE_MEASURED_PER_CLK_SM = {"u64": 3.16, "u32": 15.98}  # profiles/r01_peaks.jsonl (gold64 / shoup32)
HBM_GBS_FALLBACK = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent

WORKLOADS = {
    "C4_n20": dict(cfg="C4_n20", desc="C4 @ n=2^20: Goldilocks f-circulant matvec, batch 64, f=w^n"),
    "S1": dict(cfg="S1", desc="S1: p=998244353 f-circulant matvec n=2^20, batch 64, f=w^n"),
    "C2_f1": dict(cfg="C2_f1", desc="C2: p=998244353 circulant matvec n=2^12, batch 4096, f=1"),
    "C2_fm1": dict(cfg="C2_fm1", desc="C2: p=998244353 negacyclic matvec n=2^12, batch 4096, f=p-1"),
    **{f"C4_n{L}": dict(cfg=f"C4_n{L}", desc=f"C4 @ n=2^{L}: Goldilocks f-circulant matvec, batch 2^{26 - L}")
       for L in range(12, 23) if L != 20},
}
MMAX = {"u64": 12, "u32": 13}  # fcirc_max_fused_log2 (matvec_impl.cuh FTraits::MMAX)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
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


def algorithmic_modmuls(kind: str, n: int, batch: int, width: str) -> float:
    """Algorithmic modmuls per step attributed to one kernel kind:
    M_const = 1.5 n L (0.5 n L each for the a split, the b split, the recombination), M_var = n."""
    L = n.bit_length() - 1
    M = min(L, MMAX[width])
    K = L - M
    if kind == "k_block_fused":
        return batch * n * (1.5 * L + 1)
    if kind == "k_block_sub":
        return batch * n * (1.5 * M + 1)
    if kind == "k_cols_fwd":
        return batch * n * 1.0 * K
    if kind == "k_cols_inv":
        return batch * n * 0.5 * K
    return 0.0


def cpu_oracle_rate(inp, seconds: float = 3.0, instance: int = 0):
    """Time the oracle (as it stands) on a bounded sample: entries of one instance, O(n) each."""
    import oracle
    p, f, n = inp["p"], inp["f"], inp["n"]
    threads = oracle.default_threads()
    a, b = inp["a"][instance], inp["b"][instance]
    probe = max(threads, 32)
    t0 = time.perf_counter()
    oracle.fcirc_entries(p, f, a, b, np.arange(probe, dtype=np.int64))
    dt = time.perf_counter() - t0
    count = int(min(n, max(probe, probe * seconds / max(dt, 1e-6))))
    idx = np.random.default_rng(7).integers(0, n, count).astype(np.int64)
    t0 = time.perf_counter()
    oracle.fcirc_entries(p, f, a, b, idx)
    dt = time.perf_counter() - t0
    return count / dt, count, dt, threads


# ------------------------------------------------------------------------------------ arms

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = WORKLOADS[args.config]
    cfg = {k: v for k, v in synth.CONFIGS[w["cfg"]].items() if k != "kind"}
    inp = synth.matvec_inputs(**cfg)
    n = inp["n"]
    import oracle
    threads = oracle.default_threads()
    # each step: a bounded sample of the workload (entries of one instance), ~1 s of wall time
    rate, count, dt, _ = cpu_oracle_rate(inp, seconds=0.5)
    per_step = max(threads, int(rate * 1.0))
    times = []
    for s in range(args.warmup + args.steps):
        k = s % inp["batch"]
        idx = np.random.default_rng(100 + s).integers(0, n, per_step).astype(np.int64)
        t0 = time.perf_counter()
        oracle.fcirc_entries(inp["p"], inp["f"], inp["a"][k], inp["b"][k], idx)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * len(times) / total / 1e9
    sample = (f"{per_step} seeded-random output entries per step of one instance (step s -> instance s mod "
              f"{inp['batch']}) of {w['desc']}; Definition 2 written out, O(n) multiply-adds per entry")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg_dtype(inp["p"]),
        "data": "synthetic", "config": config_block(args, inp, w),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cfg_dtype(p: int) -> str:
    return "u64" if p >= (1 << 32) else "u32"


def config_block(args, inp, w):
    return {"workload": w["desc"], "p": int(inp["p"]), "n": int(inp["n"]), "batch": int(inp["batch"]),
            "f": "w^n" if inp.get("w") not in (None, 1) else ("1" if inp["f"] == 1 else "p-1"),
            "l2": "inputs larger than L2 (a, b, c each %.0f MiB per rank; L2 126 MB)" %
                  (inp["a"].nbytes / 2**20),
            "parallelism": f"replicas x{args.gpus} (independent instances per GPU, no collective)"}


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
    w = WORKLOADS[args.config]
    cfg = {k: v for k, v in synth.CONFIGS[w["cfg"]].items() if k != "kind"}
    inp = synth.matvec_inputs(**rank_config(cfg, rank))
    p, f, n, batch = inp["p"], inp["f"], inp["n"], inp["batch"]
    width = cfg_dtype(p)
    a = torch.from_numpy(inp["a"]).cuda()
    b = torch.from_numpy(inp["b"]).cuda()
    c = torch.empty_like(a)
    stream = torch.cuda.current_stream()

    # plan build (first call) timed separately
    t0 = time.perf_counter()
    fc.matvec(a, b, f, p, out=c)
    torch.cuda.synchronize()
    plan_ms = 1000 * (time.perf_counter() - t0)
    for _ in range(max(args.warmup - 1, 2)):
        fc.matvec(a, b, f, p, out=c)
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    fc.profile_enable(True)
    with sampler:
        ev0.record(stream)
        for _ in range(args.steps):
            fc.matvec(a, b, f, p, out=c)
            launches += fc.last_launch_count()
        ev1.record(stream)
        torch.cuda.synchronize()
    fc.profile_enable(False)
    prof = fc.profile_read()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world)
    ms_step = ms_max / args.steps
    value = whole_job_gelems(world, batch, n, args.steps, ms_max)

    # ---- roofline of the dominant kernel
    dom = max((k for k in prof if prof[k][0] > 0), key=lambda k: prof[k][1])
    cnt, kms = prof[dom]
    per_launch_mm = algorithmic_modmuls(dom, n, batch, width) * args.steps / cnt
    avg_ms = kms / cnt
    achieved = per_launch_mm / (avg_ms * 1e-3) / 1e12
    peak = SMS * SM_MHZ * 1e6 * MODMUL_PER_CLK_SM[width] / 1e12
    mp = measured_peaks()
    hbm = (mp or {}).get("hbm_gbs", HBM_GBS_FALLBACK)
    L = n.bit_length() - 1
    step_mm = batch * n * (1.5 * L + 1)
    step_bytes = 3 * batch * n * (8 if width == "u64" else 4)
    t_roof = max(step_bytes / (hbm * 1e9), step_mm / (peak * 1e12))
    roofline = {
        "bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "Tmodmul/s",
        "frac": achieved / peak, "traffic": None,
        "per_launch": {"modmuls": per_launch_mm, "avg_ms": avg_ms, "launches": cnt},
        "peak_derivation": f"{SMS} SMs x {SM_MHZ:.0f} MHz x {MODMUL_PER_CLK_SM[width]:.0f} modmul/clk/SM "
                           f"(minimal FMA-pipe slots per modmul, DESIGN.md §6)",
        "primitive_microbench_tmodmul_s": SMS * SM_MHZ * 1e6 * PRIMITIVE_MEASURED_PER_CLK_SM[width] / 1e12,
        "kernel_share_of_step": kms / ms,
        "kernels": {k: {"launches": v[0], "ms_total": v[1]} for k, v in prof.items() if v[0]},
        "step": {"t_roof_ms": 1000 * t_roof, "frac": 1000 * t_roof / ms_step,
                 "hbm_bound_ms": 1000 * step_bytes / (hbm * 1e9), "alu_bound_ms": 1000 * step_mm / (peak * 1e12),
                 "hbm_gbs_peak": hbm, "hbm_gbs_achieved_alg": step_bytes / (ms_step * 1e-3) / 1e9},
    }

    # ---- end to end through the public host API (pinned host buffers, H2D + kernels + D2H)
    e2e = None
    if not args.no_e2e:
        ha = torch.from_numpy(inp["a"]).pin_memory()
        hb = torch.from_numpy(inp["b"]).pin_memory()
        hc = torch.empty_like(ha).pin_memory()
        fc.matvec_host(ha, hb, f, p, out=hc)
        if world > 1:
            dist.barrier()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            fc.matvec_host(ha, hb, f, p, out=hc)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        esz = 8 if width == "u64" else 4
        e2e = {"value": world * batch * n * e_steps / dt / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * batch * n * esz, "d2h_bytes_per_step": batch * n * esz,
               "steps": e_steps, "api": "fcirc_matvec_host (pinned host buffers; wall clock, synchronous call)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, count, dt, threads = cpu_oracle_rate(inp, seconds=args.cpu_seconds)
        cpu = {"value": rate / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{count} seeded-random output entries of instance 0 of {w['desc']} "
                         f"(Definition 2, O(n) multiply-adds each); {dt:.1f} s wall"}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": width, "data": "synthetic (seeded uniform residues, SURVEY §8(d))",
            "config": config_block(args, inp, w), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": sampler.summary(), "plan_build_ms": plan_ms,
        }
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_fcirc(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/: launch lists (per-kernel shares) and --set full reports
(key counters per kernel).  Usage:
  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py full <report.ncu-rep | raw.csv>   (raw.csv: ncu -i R --page raw --csv)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki].split("(")[0]][0] += 1
        agg[r[ki].split("(")[0]][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list {path}: gpu__time_duration.sum per kernel (cold-cache, serialised)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:72]:72s} launches={c:5d} total_us={t / 1e3:10.1f} avg_us={t / c / 1e3:8.1f} share={t / tot:.3f}")


def full(path):
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"## {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {units[hdr.index(k)]}")


UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20, "GB": 1 << 30}


def traffic(path, kind, workload, kernel_regex, out_json="profiles/traffic.json"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernels matching
    kernel_regex in an ncu --set full report -> profiles/traffic.json[workload][kind]
    (read by bench.py for the roofline "traffic" field)."""
    import json
    import os
    import re
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    vals = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if not re.search(kernel_regex, d.get("Kernel Name", "")):
            continue
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = units[hdr.index(k)]
            tot += float(d[k].replace(",", "")) * UNIT_SCALE.get(u, 1)
        vals.append(tot)
    if not vals:
        raise SystemExit(f"no kernel matching {kernel_regex!r} in {path}")
    db = json.load(open(out_json)) if os.path.exists(out_json) else {}
    db.setdefault(workload, {})[kind] = {
        "bytes_per_launch": sum(vals) / len(vals), "launches_captured": len(vals), "report": path,
        "note": "ncu --set full (default --cache-control all: L2 flushed before each replay, so "
                "intermediates the pipeline keeps in L2 are counted as DRAM reads)"}
    json.dump(db, open(out_json, "w"), indent=1, sort_keys=True)
    print(json.dumps(db[workload][kind]))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "traffic":
        traffic(*sys.argv[2:])
    else:
        {"launches": launches, "full": full}[cmd](sys.argv[2])

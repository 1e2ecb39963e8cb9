#!/usr/bin/env python
"""Print DESIGN.md §10's results table from a set of committed bench lines (dev tool).

usage: design_table.py PREFIX      e.g. profiles/r02z_bench_
"""
import json
import sys

ORDER = ["C4n20", "C4_n12", "C4_n14", "C4_n16", "C4_n18", "C4_n22", "S1", "C2_f1", "C2_fm1", "C1", "C3", "C5",
         "S2_n512", "N3_gold", "N3_u32"]
NAMES = {"C4n20": "**C4 n=2^20 (headline)**", "C4_n12": "C4 n=2^12", "C4_n14": "C4 n=2^14", "C4_n16": "C4 n=2^16",
         "C4_n18": "C4 n=2^18", "C4_n22": "C4 n=2^22", "S1": "S1 u32 n=2^20", "C2_f1": "C2 f=1", "C2_fm1": "C2 f=p−1",
         "C1": "C1 n=2^10, batch 1 (graph)", "C3": "C3 polymul (circulant entries)",
         "C5": "C5 bigint (output limb positions, graph)", "S2_n512": "S2 n=512 (paper ring, its own product rate)",
         "N3_gold": "N3 any-n n=1000003, Goldilocks (outputs)", "N3_u32": "N3 any-n n=1000003, u32 (outputs)"}


def f(x, n=3):
    try:
        return f"{float(x):.{n}f}"
    except (TypeError, ValueError):
        return "—"


def main():
    pre = sys.argv[1]
    print("| config | Gelem/s | ms/step (mean) | ms min | dominant kernel | achieved Tmodmul/s | frac | ceil | step "
          "| e2e Gelem/s | cpu Gelem/s | par |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for k in ORDER:
        try:
            d = json.load(open(f"{pre}{k}.json"))
        except OSError:
            continue
        r = d["roofline"]
        v = f"{d['value']:.2f}"
        if k == "C4n20":
            v = f"**{v}**"
        lat = k == "C1"   # latency-bound single product: no meaningful roofline fraction
        print(f"| {NAMES[k]} | {v} | {d['ms_per_step']:.4f} | {d.get('ms_min', float('nan')):.4f} | {r.get('kernel', '—')} "
              f"| {'—' if lat else f(r.get('achieved'))} | {'—' if lat else f(r.get('frac'))} "
              f"| {'—' if lat else f(r.get('frac_vs_ceiling'))} | {'—' if lat else f(r['step'].get('frac'))} "
              f"| {d['e2e']['value']:.2f} | {d['cpu_baseline']['value']:.2e} | {d['parity']['mismatches']} |")


if __name__ == "__main__":
    main()

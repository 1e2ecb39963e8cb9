#!/usr/bin/env python
"""Summarise an ncu `--page source --csv --print-source sass` export (dev tool, no GPU).

usage: ncu_src_stalls.py <csv> [top]

Prints the kernel's stall-reason shares (warp-state samples), the samples per opcode, and the `top`
instructions by samples with their leading stall reasons.
"""
import csv
import sys
from collections import Counter, defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    if not hdr:
        sys.exit("no source table")
    h = rows[hdr[0]]
    end = hdr[1] - 1 if len(hdr) > 1 else len(rows)
    data = [r for r in rows[hdr[0] + 1:end] if len(r) >= len(h)]
    ci = {k: i for i, k in enumerate(h)}
    cols = [c for c in h if c.startswith("stall_") and "(Not" not in c]
    tot = Counter()
    per_op = defaultdict(Counter)
    samples = []
    for r in data:
        src = r[ci["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        base = op.split(".")[0]
        n = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        st = {c: float(r[ci[c]] or 0) for c in cols}
        tot.update(st)
        per_op[base].update({"samples": n})
        samples.append((n, src, st))
    s = sum(tot.values()) or 1
    print("stall shares:", ", ".join(f"{c[6:]} {v / s * 100:.1f}%" for c, v in tot.most_common(10)))
    ops = sorted(per_op.items(), key=lambda kv: -kv[1]["samples"])
    print("samples by opcode:", ", ".join(f"{k} {v['samples'] / s * 100:.1f}%" for k, v in ops[:14]))
    samples.sort(key=lambda x: -x[0])
    for n, src, st in samples[:top]:
        lead = ", ".join(f"{c[6:]} {v:.0f}" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{n:8.0f}  {src[:58]:58s} {lead}")


if __name__ == "__main__":
    main()

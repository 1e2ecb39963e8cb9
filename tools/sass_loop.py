#!/usr/bin/env python
"""Histogram the SASS of the innermost backward-branch loop of a kernel (dev tool).
usage: sass_loop.py <binary> <kernel-substring> [ops_per_iteration]"""
import re
import subprocess
import sys
from collections import Counter

binary, pat = sys.argv[1], sys.argv[2]
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = [f for f in funcs if pat in f.split("\n")[0]][0]
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# find the last backward branch
loop = None
for addr, txt in ins:
    m = re.search(r"BRA\s+(?:`?\(?\.L_x_\d+\)?|0x([0-9a-f]+))", txt)
    t = re.search(r"0x([0-9a-f]+)", txt) if "BRA" in txt else None
    if "BRA" in txt and t and int(t.group(1), 16) < addr:
        loop = (int(t.group(1), 16), addr)
if loop is None:
    print("no backward branch; whole kernel")
    sel = ins
else:
    sel = [x for x in ins if loop[0] <= x[0] <= loop[1]]
ops = Counter()
for _, txt in sel:
    op = re.sub(r"^@!?U?P\w+\s+", "", txt).split()[0]
    ops[op] += 1
fma = {"IMAD", "IMAD.X", "IMAD.MOV.U32", "IMAD.MOV", "IMAD.IADD", "IMAD.U32", "IMAD.SHL.U32", "HFMA2", "FFMA", "IMAD.WIDE.U32",
       "IMAD.WIDE", "IMAD.HI.U32", "IMAD.HI"}
heavy2 = {"IMAD.WIDE.U32", "IMAD.WIDE", "IMAD.HI.U32", "IMAD.HI"}
tot = sum(ops.values())
fma_slots = sum(c * (2 if o in heavy2 else 1) for o, c in ops.items() if o in fma)
alu = sum(c for o, c in ops.items() if o.split(".")[0] in ("IADD3", "LOP3", "SEL", "ISETP", "SHF", "LEA", "PRMT", "VIADD", "IMNMX", "VIMNMX", "MOV", "P2R", "R2P", "PLOP3", "FSEL", "ISETP"))
print(f"loop {loop}: {tot} instr, per op {tot / per:.1f}; FMA-pipe slots {fma_slots / per:.1f}, ALU {alu / per:.1f}")
for o, c in ops.most_common(25):
    print(f"  {o:22s} {c:5d}  {c / per:6.2f}")

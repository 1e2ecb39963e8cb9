#!/usr/bin/env python
"""Classify the SASS of a kernel by issue pipe (dev tool; no GPU needed).

usage: sass_pipes.py <binary> <kernel-substring> [divisor] [--loop]

--loop restricts the count to the body of the last backward branch (a microbenchmark's loop).

Counts every instruction of the function in the ALU pipe (IADD3, LOP3, SEL, ISETP, LEA, SHF,
PLOP3, P2R, IMNMX, ...), the FMA pipe (IMAD*, incl. IMAD.WIDE / .HI / .X / .MOV / .IADD), memory
and other, optionally divided by `divisor` (e.g. butterflies in the loop body).  Used to steer the
Goldilocks helpers of csrc/modarith.cuh toward a balanced ALU/FMA mix.
"""
import re
import subprocess
import sys
from collections import Counter

ALU = ("IADD3", "LOP3", "SEL", "ISETP", "LEA", "SHF", "PLOP3", "P2R", "R2P", "IMNMX", "VIMNMX", "IABS",
       "FLO", "POPC", "BREV", "PRMT", "MOV", "ISCADD", "VIADD", "IADD")
FMA = ("IMAD",)
MEM = ("LDG", "STG", "LDS", "STS", "LDC", "LDCU", "LDL", "STL", "ATOM", "RED", "LD", "ST", "LDGSTS")


def classify(op: str) -> str:
    base = op.split(".")[0]
    if base in FMA:
        return "fma"
    if base in MEM:
        return "mem"
    if base in ALU:
        return "alu"
    if base.startswith("U"):
        return "uniform"
    return "other"


def main():
    args = [a for a in sys.argv[1:] if a != "--loop"]
    loop_only = "--loop" in sys.argv
    binary, pat = args[0], args[1]
    div = float(args[2]) if len(args) > 2 else 1.0
    sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    body = [f for f in funcs if pat in f.split("\n")[0]]
    if not body:
        sys.exit(f"no function matching {pat}")
    ins = []
    for line in body[0].split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*)", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    if loop_only:
        lo = None
        for addr, op, rest in ins:
            t = re.search(r"0x([0-9a-f]+)", rest)
            if op.startswith("BRA") and t and int(t.group(1), 16) < addr:
                lo = (int(t.group(1), 16), addr)
        if lo:
            ins = [x for x in ins if lo[0] <= x[0] <= lo[1]]
    ops = [op for _, op, _ in ins]
    pipes = Counter(classify(o) for o in ops)
    print(f"{body[0].split(chr(10))[0][:90]}")
    print("  " + "  ".join(f"{k}={v / div:.2f}" for k, v in sorted(pipes.items())))
    top = Counter(ops).most_common(14)
    print("  " + "  ".join(f"{k}:{v / div:.2f}" for k, v in top))


if __name__ == "__main__":
    main()

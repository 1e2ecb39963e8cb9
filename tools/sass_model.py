#!/usr/bin/env python
"""Per-warp pipe-cycle model of each kernel in a binary (dev tool; no GPU needed).

usage: sass_model.py <binary> [name-substring ...]

Static SASS of each matching function, classified with the pipe costs calibrated against the
r01n ncu capture of k_block<FieldGold,12,8> (profiles/r01n_ncu_raw_C4n20.csv: fmaheavy 76 %,
alu 66 %, issue 65 % reproduced within 1 %):
  fmaheavy: IMAD.WIDE*, IMAD.HI* = 4 cycles per warp instruction; every other IMAD* and VIADD = 2
  alu:      IADD3, LOP3, SEL, ISETP, LEA, SHF, MOV, PRMT, ... = 2
  issue:    1 per instruction
bound = max(fma, alu, issue) cycles per warp (straight-line code: what each thread executes once).
"""
import re
import subprocess
import sys

ALU = ("IADD3", "LOP3", "SEL", "ISETP", "LEA", "SHF", "PLOP3", "P2R", "R2P", "IMNMX", "VIMNMX", "IABS",
       "FLO", "POPC", "BREV", "PRMT", "MOV", "ISCADD", "IADD", "CS2R")


def model(lines):
    fma = alu = n = 0
    wide = 0
    for op in lines:
        base = op.split(".")[0]
        n += 1
        if base == "IMAD":
            if ".WIDE" in op or ".HI" in op:
                fma += 4
                wide += 1
            else:
                fma += 2
        elif base == "VIADD":
            fma += 2
        elif base in ALU:
            alu += 2
    return n, wide, fma, alu


def main():
    binary, pats = sys.argv[1], sys.argv[2:]
    sass = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s*Function : ", sass)[1:]:
        name = f.split("\n")[0].strip()
        if pats and not all(p in name for p in pats):
            continue
        ops = re.findall(r"^\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f, re.M)
        n, wide, fma, alu = model(ops)
        print(f"{name[:90]:90s} n={n:5d} wide={wide:4d} fma={fma:5d} alu={alu:5d} bound={max(fma, alu, n):5d}")


if __name__ == "__main__":
    main()

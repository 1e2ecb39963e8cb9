#!/usr/bin/env python
"""Bank-conflict model of the staged-twiddle loads of the 32-bit k_block (M = 12, R = 8; dev tool, CPU
only): for every phase, level, butterfly slot and warp, the 8-byte twiddle indices the 32 lanes load,
mapped through a candidate layout, counted in wavefronts (tools/bank_model.py) against the minimum."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bank_model import Phases, wavefronts
M, R = 12, 8
P = Phases(M, R, True)
def twidx(ph, t, s0, jb):
    x = P.ins_t(ph, t) | P.cslot(ph, s0)
    bit = P.lo(ph) + jb
    return (1 << (M - 1 - bit)) | (x >> (bit + 1))
layouts = {
  'identity': lambda i: i,
  'xor_swz (current)': lambda i: i ^ ((i >> 4) & 31),
  'pad1/16': lambda i: i + (i >> 4),
  'pad1/32': lambda i: i + (i >> 5),
  'pad2/32': lambda i: i + 2 * (i >> 5),
  'pad1/8': lambda i: i + (i >> 3),
}
for name, f in layouts.items():
    tot = ideal = 0
    for ph in range(P.NPH):
        for jb in range(P.rp(ph)):
            for s0 in range(R):
                if (s0 >> jb) & 1: continue
                for w in range(P.T // 32):
                    addrs = [f(twidx(ph, w * 32 + l, s0, jb)) for l in range(32)]
                    tot += wavefronts(addrs, 8)
                    # ideal: distinct addresses / 16 per wavefront, at least 1 per half
                    d = [len(set(addrs[:16])), len(set(addrs[16:]))]
                    ideal += sum(max(1, (x * 2 + 31) // 32) for x in d)
    print(f"{name:22s} wavefronts {tot} ratio {tot/ideal:.3f}")

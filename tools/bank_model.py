#!/usr/bin/env python
"""Shared-memory bank-conflict model of k_block's phase exchanges (dev tool, CPU only).

Replays the address pattern of csrc/fcirc_kernels.cuh (Phases<NB, R>::ins_t / cslot) for every
phase, slot and warp, applies a candidate layout function and counts wavefronts per warp access:
4-byte elements -> 32 banks per warp request, 8-byte elements -> two 16-thread wavefronts.
Prints the ratio to the conflict-free count (1.00 = conflict-free) for the former padded layout
and the swizzle x ^ ((x >> r) & MASK) with the short phase on top (the current kernels).

usage: python tools/bank_model.py
"""


def ilog2(x):
    return x.bit_length() - 1


class Phases:
    def __init__(self, NB, R, short_first=True):
        self.NB, self.R, self.r = NB, R, ilog2(R)
        self.T = (1 << NB) // R
        self.NPH = 0 if NB == 0 else (NB + self.r - 1) // self.r
        self.short_first = short_first

    def rp(self, ph):
        short = self.NB - self.r * (self.NPH - 1)
        if self.short_first:
            return short if ph == 0 else self.r
        return self.r if ph < self.NPH - 1 else short

    def lo(self, ph):
        return self.NB - sum(self.rp(i) for i in range(ph + 1))

    def ins_t(self, ph, t):
        l, w = self.lo(ph), self.rp(ph)
        return ((t >> l) << (l + w)) | (t & ((1 << l) - 1))

    def cslot(self, ph, s):
        l, w = self.lo(ph), self.rp(ph)
        j, g = s & ((1 << w) - 1), s >> w
        u = g * self.T
        return ((u >> l) << (l + w)) | (j << l) | (u & ((1 << l) - 1))


def wavefronts(addrs, esz):
    groups = [addrs] if esz == 4 else [addrs[:16], addrs[16:]]
    tot = 0
    for g in groups:
        banks = {}
        for a in g:
            for k in range(esz // 4):
                w = a * (esz // 4) + k
                banks.setdefault(w % 32, set()).add(w)
        tot += max(len(v) for v in banks.values()) if banks else 0
    return tot


def ratio(NB, R, esz, layout, short_first):
    P = Phases(NB, R, short_first)
    tot = ideal = 0
    for ph in range(P.NPH):
        for s in range(R):
            for w0 in range(0, P.T, 32):
                n = min(32, P.T - w0)
                ad = [layout(P.ins_t(ph, t) + P.cslot(ph, s)) for t in range(w0, w0 + n)]
                tot += wavefronts(ad, esz)
                ideal += 1 if esz == 4 else (2 if n > 16 else 1)
    return tot / ideal if ideal else 1.0


def ratio_cols(K, R, W, esz, rowmap, short_first):
    """k_cols: W consecutive columns per CTA, thread (c = tid % W, t = tid / W), smem rows of W."""
    P = Phases(K, R, short_first)
    tot = ideal = 0
    nthr = W * P.T
    for ph in range(P.NPH):
        for s in range(R):
            for w0 in range(0, nthr, 32):
                ad = []
                for tid in range(w0, min(w0 + 32, nthr)):
                    c, t = tid % W, tid // W
                    ad.append(rowmap(P.ins_t(ph, t) + P.cslot(ph, s)) * W + c)
                tot += wavefronts(ad, esz)
                ideal += 1 if esz == 4 else 2
    return tot / ideal


def ratio_twiddles(M, R, swz):
    """k_block with staged twiddles: LDS.64 of the twiddle of each butterfly (local heap index)."""
    P = Phases(M, R, True)
    tot = ideal = 0
    for ph in range(P.NPH):
        rp, lo = P.rp(ph), P.lo(ph)
        for l in range(rp):
            bbit = lo + rp - 1 - l
            for s0 in range(R):
                if (s0 >> (rp - 1 - l)) & 1:
                    continue
                for w0 in range(0, P.T, 32):
                    ad = sorted({swz((1 << (M - 1 - bbit)) - 1 + ((P.ins_t(ph, t) | P.cslot(ph, s0)) >> (bbit + 1)))
                                 for t in range(w0, min(w0 + 32, P.T))})
                    tot += wavefronts(ad, 8) if len(ad) > 1 else 1
                    ideal += 1 if len(ad) <= 16 else 2
    return tot / ideal


def main():
    for esz, sh, mask in [(4, 5, 31), (8, 4, 15)]:
        for R in (4, 8, 16):
            r = ilog2(R)
            cells = []
            for NB in range(5, 14):
                if (1 << NB) // R > 1024:
                    continue
                pad = ratio(NB, R, esz, lambda x: x + (x >> sh), False)
                swz = ratio(NB, R, esz, lambda x: x ^ ((x >> r) & mask), True)
                cells.append(f"M{NB}:{pad:.2f}/{swz:.2f}")
            print(f"{esz}B R={R:2d} pad/swizzle  " + " ".join(cells))
    print("k_cols (rows of W columns): (row + row>>4) pad / row ^ ((row >> r) & 7) swizzle")
    for esz in (4, 8):
        for R in (8, 16):
            r = ilog2(R)
            cells = []
            for K in range(6, 11):
                W = max(8, (256 * R) >> K)
                if W * (1 << K) // R > 1024:
                    continue
                old = ratio_cols(K, R, W, esz, lambda x: x + (x >> 4), False)
                new = ratio_cols(K, R, W, esz, lambda x: x ^ ((x >> r) & 7), True)
                cells.append(f"K{K}/W{W}:{old:.2f}/{new:.2f}")
            print(f"{esz}B R={R:2d} " + " ".join(cells))
    print("k_block staged twiddles (8 B): plain index / i ^ ((i >> 4) & 31)")
    for M, R in [(11, 8), (12, 8), (13, 8), (12, 16)]:
        print(f"M{M} R={R}: {ratio_twiddles(M, R, lambda i: i):.2f} / "
              f"{ratio_twiddles(M, R, lambda i: i ^ ((i >> 4) & 31)):.2f}")


if __name__ == "__main__":
    main()

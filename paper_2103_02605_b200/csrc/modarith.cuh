// modarith.cuh — ring arithmetic of the hot path.
//
// The paper works in "a ring R" (Theorem 1) and, for its own CPU experiment, in
// Z/pZ[sqrt 3] with p = 2^31-1 using 64-bit Java longs.  On B200 the ring is Z/p for
// NTT-friendly primes, with the integer pipes in mind (measured, profiles/r01_peaks.jsonl):
// IMAD 64/clk/SM, IMAD.HI and IMAD.WIDE 32/clk/SM, IADD3/LOP3 64/clk/SM.
//
//  * FieldU32: p < 2^30 (998244353, 469762049, 167772161), 4p < 2^32.
//      const x var  : Shoup (twiddle w with q = floor(w 2^32 / p)): 1 IMAD.HI + 2 IMAD, out [0,2p)
//      var x var    : Montgomery REDC with R = 2^32, out [0,2p) (leaves only)
//      lazy ranges  : forward butterflies keep values in [0,4p), inverse ones in [0,2p)
//  * FieldGold: p = 2^64 - 2^32 + 1.  Values are kept "weakly reduced" in [0, 2^64).
//      64x64 -> 128 with IMAD.WIDE chains; const x var (twiddles, stored times 2^64 mod p) by a
//      Montgomery reduction with R = 2^64 (8 add/sub, p^-1 = 1 + 2^32 mod 2^64); var x var
//      (leaves) by the special reduction 2^64 == 2^32 - 1 (=: EPS), 2^96 == -1 (mod p).
//
// The in-place form of Algorithm 1 used by the kernels:
//   forward (row a)   : (x, y) -> (x + s y, x - s y)      [rows of A_M1 and A_M2, P:66-67]
//   forward (vector b): (x, y) -> (s x + y, s x - y)      [b1 sqrt f +- b2, P:66-67]
//   leaf              : M = a^ b^                          [1x1 product]
//   inverse           : (M1, M2) -> ((M1 + M2) s^-1, M1 - M2)   [c1 = (M1+M2)/(2 sqrt f),
//                        c2 = (M1+M2)/2 - M2 = (M1-M2)/2, with every 1/2 deferred]
//   last inverse level: both outputs also multiplied by K = n^-1 (x R for Montgomery leaves),
//                        which absorbs the L deferred factors 1/2.
#pragma once
#include <cstdint>

namespace fcirc {

// Programmatic dependent launch (PDL; launch attribute set unless FCIRC_PDL=0): every kernel of the path starts by
// waiting for the previous kernel in the stream to complete (griddepcontrol.wait: all of its memory
// visible) and then allows the next one to be scheduled (griddepcontrol.launch_dependents), so the
// next kernel's CTAs fill the SMs freed during this kernel's last wave instead of waiting for a new
// launch.  Both are no-ops for launches without the PDL attribute.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// 32-bit NTT primes
// ------------------------------------------------------------------------------------------
struct __align__(8) TwU32 {  // 8-byte aligned: one 64-bit load per twiddle
  uint32_t w, q;  // twiddle and its Shoup quotient floor(w * 2^32 / p)
};

struct FieldU32 {
  using T = uint32_t;
  using Tw = TwU32;
  uint32_t p;         // modulus
  uint32_t p2;        // 2p
  uint32_t pinv_neg;  // -p^-1 mod 2^32 (Montgomery)

  // x * w mod p, result in [0, 2p) for any x < 2^32 (Shoup / Harvey)
  __device__ __forceinline__ uint32_t mulc(uint32_t x, TwU32 t) const {
    uint32_t hq = __umulhi(x, t.q);
    return x * t.w - hq * p;
  }
  // [0, 4p) -> [0, 2p)
  __device__ __forceinline__ uint32_t red2(uint32_t x) const { return min(x, x - p2); }
  // [0, 2p) -> [0, p)
  __device__ __forceinline__ uint32_t red1(uint32_t x) const { return min(x, x - p); }

  __device__ __forceinline__ void fwd_a(uint32_t& x, uint32_t& y, TwU32 s) const {
    uint32_t X = red2(x);
    uint32_t t = mulc(y, s);
    x = X + t;
    y = X - t + p2;
  }
  static constexpr bool NEG_B = false;   // see FieldGold::fwd_bn
  __device__ __forceinline__ void fwd_bn(uint32_t& x, uint32_t& y, TwU32 s) const { fwd_b(x, y, s); }
  __device__ __forceinline__ void fwd_b(uint32_t& x, uint32_t& y, TwU32 s) const {
    uint32_t t = mulc(x, s);
    uint32_t Y = red2(y);
    x = t + Y;
    y = t - Y + p2;
  }
  // inputs in [0, 2p), outputs in [0, 2p)
  __device__ __forceinline__ void inv(uint32_t& u, uint32_t& v, TwU32 si) const {
    uint32_t s = u + v;
    uint32_t d = u - v + p2;
    u = mulc(s, si);
    v = red2(d);
  }
  // global level 0: outputs canonical [0, p); si_k = s^-1 K, k = K
  __device__ __forceinline__ void inv_last(uint32_t& u, uint32_t& v, TwU32 si_k, TwU32 k) const {
    uint32_t s = u + v;
    uint32_t d = u - v + p2;
    u = red1(mulc(s, si_k));
    v = red1(mulc(d, k));
  }
  // leaves: inputs in [0, 4p); returns a b R^-1 mod p in [0, 2p).  Lazy: only a is brought to
  // [0, 2p), so T = a b < 8 p^2 < 2^64 (p < 2^30) and (T + m p) / 2^32 < p (8 p / 2^32 + 1) < 2.9 p
  // fits 32 bits; one red2 returns it to [0, 2p) (4 range corrections fewer than reducing both
  // factors to [0, p) first: 10 instead of 14 instructions per leaf).
  __device__ __forceinline__ uint32_t leaf(uint32_t a, uint32_t b) const {
    a = red2(a);
    uint32_t lo = a * b;
    uint32_t hi = __umulhi(a, b);
    uint32_t m = lo * pinv_neg;
    // (a b + m p) / 2^32: the low words cancel exactly (lo + m p == 0 mod 2^32); carry = (lo != 0)
    uint32_t mh = __umulhi(m, p);
    return red2(hi + mh + (lo != 0u));
  }
  // n = 1: c = a b exactly; k = K (= R mod p) undoes the Montgomery factor
  __device__ __forceinline__ uint32_t single(uint32_t a, uint32_t b, TwU32 k) const {
    return red1(mulc(leaf(a, b), k));
  }
};

// ------------------------------------------------------------------------------------------
// Goldilocks p = 2^64 - 2^32 + 1
// ------------------------------------------------------------------------------------------
struct FieldGold {
  using T = uint64_t;
  using Tw = uint64_t;
  static constexpr uint64_t P = 0xFFFFFFFF00000001ull;
  static constexpr uint64_t EPS = 0xFFFFFFFFull;  // 2^64 mod p

  // All helpers work on 32-bit halves with explicit PTX carry chains.  The wrap-around corrections
  // (+-EPS when a 64-bit add/sub carried/borrowed, and the final r >= p test of a reduction) are
  // written the way that measured fewest SASS instructions: after an add chain, the carry becomes
  // a predicate and the correction two predicated adds (add_c, reduce4: ptxas emits ISETP + @P
  // VIADD instead of computing both alternatives and selecting with an IMAD.MOV, -8 % instructions
  // per butterfly, profiles/r01k_sweep_gold_predicated_ab.txt); after a subtract chain
  // `subc.u32 m, 0, 0` yields m = -borrow (0 or 0xffffffff = EPS's low word) and the correction is
  // one more subtract chain (sub_c, sub_w).  (PTX carry flags are the hardware carry: after an add,
  // `subc m, 0, 0` gives carry - 1, NOT -carry, so add and subtract chains are never mixed;
  // tests/test_modarith_ptx.py executes every chain under that model.)
  __device__ __forceinline__ static uint32_t lo32(uint64_t x) { return (uint32_t)x; }
  __device__ __forceinline__ static uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }
  __device__ __forceinline__ static uint64_t mk(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }

  // a + b mod p for a any 64-bit value and b < p (canonical): on a carry out of 2^64 add EPS
  // (= lo - 1, with a carry into hi unless lo == 0); a + b - 2^64 + EPS <= 2^64 - 2: no second
  // carry.  Weak result.
  __device__ __forceinline__ static uint64_t add_c(uint64_t a, uint64_t b) {
    uint32_t s0, s1;
    asm("{\n\t.reg .u32 c;\n\t.reg .pred p, q;\n\t"
        "add.cc.u32  %0, %2, %4;\n\t"
        "addc.cc.u32 %1, %3, %5;\n\t"
        "addc.u32    c, 0, 0;\n\t"
        "setp.ne.u32 p, c, 0;\n\t"              // carry out of 2^64: + EPS
        "setp.ne.and.u32 q, %0, 0, p;\n\t"      // ... which carries into hi unless lo == 0
        "@p sub.u32  %0, %0, 1;\n\t"
        "@q add.u32  %1, %1, 1;\n\t"
        "}"
        : "=&r"(s0), "=&r"(s1) : "r"(lo32(a)), "r"(hi32(a)), "r"(lo32(b)), "r"(hi32(b)));
    return mk(s0, s1);
  }
  // a - b mod p for a any 64-bit value and b < p: on a borrow subtract EPS; the wrapped value is
  // a - b + 2^64 >= 2^64 - p + 1 > EPS, so no second borrow.  Canonical if a is canonical.
  __device__ __forceinline__ static uint64_t sub_c(uint64_t a, uint64_t b) {
    uint32_t d0, d1;
    asm("{\n\t.reg .u32 m;\n\t"
        "sub.cc.u32  %0, %2, %4;\n\t"
        "subc.cc.u32 %1, %3, %5;\n\t"
        "subc.u32    m, 0, 0;\n\t"        // m = -borrow
        "sub.cc.u32  %0, %0, m;\n\t"      // - EPS
        "subc.u32    %1, %1, 0;\n\t"
        "}"
        : "=&r"(d0), "=&r"(d1) : "r"(lo32(a)), "r"(hi32(a)), "r"(lo32(b)), "r"(hi32(b)));
    return mk(d0, d1);
  }
  // a - b mod p for any 64-bit a, b: up to two borrow corrections (the second only if
  // b > a + p - 2^64 + EPS, i.e. both were large); result a - b + {0, p, 2p}, weakly reduced.
  __device__ __forceinline__ static uint64_t sub_w(uint64_t a, uint64_t b) {
    uint32_t d0, d1;
    asm("{\n\t.reg .u32 m;\n\t"
        "sub.cc.u32  %0, %2, %4;\n\t"
        "subc.cc.u32 %1, %3, %5;\n\t"
        "subc.u32    m, 0, 0;\n\t"
        "sub.cc.u32  %0, %0, m;\n\t"
        "subc.cc.u32 %1, %1, 0;\n\t"
        "subc.u32    m, 0, 0;\n\t"
        "sub.cc.u32  %0, %0, m;\n\t"
        "subc.u32    %1, %1, 0;\n\t"
        "}"
        : "=&r"(d0), "=&r"(d1) : "r"(lo32(a)), "r"(hi32(a)), "r"(lo32(b)), "r"(hi32(b)));
    return mk(d0, d1);
  }
  // (t0 + t1 2^32 + t2 2^64 + t3 2^96) mod p, canonical, with 2^64 == EPS and 2^96 == -1:
  //   V = (t1:t0) + t2 EPS - t3 as a 3-word signed value c 2^64 + (r1:r0), c in {-1, 0, 1}
  //       (V in (-2^32, 2^65 - 2^33]); (t1:t0) + t2 EPS is ONE IMAD.WIDE.U32 with carry out
  //       (mul.wide.u32 + add.cc.u64; the former mad.lo.cc / madc.hi.cc pair compiled to
  //       IMAD.IADD + IMAD.HI + a register-pair move: k_block -1.6 %, k_cols_inv2 -3.6 %,
  //       profiles/r02a_gold_ab_reduce_variants.txt);
  //   r += c EPS  (as a 64-bit two's-complement add of (c >> 31 : -c)); for c = +1 the result is
  //       <= 2^64 - 2^32 - 1 < p, for c = -1 it is in [p - EPS, p), no further wrap;
  //   canonicalise: r >= p only if r_hi == 0xffffffff and r_lo != 0, and then r - p = (r_lo - 1, 0).
  __device__ __forceinline__ static uint64_t reduce4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 c, m, h;\n\t.reg .u64 T, E, R;\n\t.reg .pred p, q;\n\t"
        "mov.b64         T, {%2, %3};\n\t"
        "mul.wide.u32    E, %4, 0xffffffff;\n\t"
        "add.cc.u64      R, T, E;\n\t"
        "addc.u32        c, 0, 0;\n\t"
        "mov.b64         {%0, %1}, R;\n\t"
        "sub.cc.u32      %0, %0, %5;\n\t"
        "subc.cc.u32     %1, %1, 0;\n\t"
        "subc.u32        c, c, 0;\n\t"
        "neg.s32         m, c;\n\t"
        "shr.s32         h, c, 31;\n\t"
        "add.cc.u32      %0, %0, m;\n\t"
        "addc.u32        %1, %1, h;\n\t"
        "setp.eq.u32     p, %1, 0xffffffff;\n\t"  // r >= p  <=>  r_hi == 2^32-1 and r_lo != 0
        "setp.ne.and.u32 q, %0, 0, p;\n\t"
        "@q sub.u32      %0, %0, 1;\n\t"          // r - p = (r_lo - 1, 0)
        "@q mov.u32      %1, 0;\n\t"
        "}"
        : "=&r"(r0), "=&r"(r1) : "r"(t0), "r"(t1), "r"(t2), "r"(t3));
    return mk(r0, r1);
  }
  // 64 x 64 -> 128 -> canonical residue in [0, p), for any 64-bit a, b (the leaves: var x var).
  __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) {
    // ptxas expands mul.lo.u64 / mul.hi.u64 into IMAD.WIDE.U32 chains with carry predicates
    const uint64_t lo = a * b, hi = __umul64hi(a, b);
    return reduce4(lo32(lo), hi32(lo), lo32(hi), hi32(hi));
  }
  // Montgomery reduction with R = 2^64 (round 3 of the arithmetic): T 2^-64 mod p, canonical, for
  // T = (t3:t2:t1:t0) with xh = (t3:t2) <= p - 2, i.e. for every product x * s with x < 2^64 and
  // s < p (T <= (2^64 - 1)(p - 1) < (p - 1) 2^64).
  //   p^-1 mod 2^64 = 1 + 2^32, so m = xl p^-1 mod 2^64 = (t0, a1) with a1 = t0 + t1 (mod 2^32),
  //   e = carry of t0 + t1; (T - m p) / 2^64 = xh - (m - a1 - e) = (xh + a1 + e) - m, a value in
  //   (-p, p) (m p <= (2^64 - 1) p and m p == xl mod 2^64); xh + a1 + e <= p - 2 + 2^32 < 2^64 (no
  //   overflow); a borrow means the value is negative and adding p = subtracting EPS mod 2^64.
  // Eight 32-bit add/sub with carry and no multiply (reduce4: one IMAD.WIDE + 13), and the result
  // needs no canonicalisation.  The twist-table entries and scaling constants are stored times
  // R mod p (= EPS) so that mulm(x, s R) = x s (api.cu: Montgomery form of the Goldilocks plan).
  __device__ __forceinline__ static uint64_t mont_reduce(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 a1, x0, x1, m;\n\t"
        "add.cc.u32  a1, %3, %2;\n\t"     // a1 = t0 + t1, CF = e
        "addc.cc.u32 x0, %4, a1;\n\t"     // x = xh + a1 + e
        "addc.u32    x1, %5, 0;\n\t"
        "sub.cc.u32  %0, x0, %2;\n\t"     // r = x - m, m = (t0, a1)
        "subc.cc.u32 %1, x1, a1;\n\t"
        "subc.u32    m, 0, 0;\n\t"        // m = -borrow
        "sub.cc.u32  %0, %0, m;\n\t"      // on a borrow: r - EPS = r + p (mod 2^64)
        "subc.u32    %1, %1, 0;\n\t"
        "}"
        : "=&r"(r0), "=&r"(r1) : "r"(t0), "r"(t1), "r"(t2), "r"(t3));
    return mk(r0, r1);
  }
  // -(T 2^-64) mod p, canonical, same precondition: the subtraction's operands swapped, m - x, again
  // a value in (-p, p) that a borrow corrects by + p
  __device__ __forceinline__ static uint64_t mont_reduce_neg(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3) {
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 a1, x0, x1, m;\n\t"
        "add.cc.u32  a1, %3, %2;\n\t"     // a1 = t0 + t1, CF = e
        "addc.cc.u32 x0, %4, a1;\n\t"     // x = xh + a1 + e
        "addc.u32    x1, %5, 0;\n\t"
        "sub.cc.u32  %0, %2, x0;\n\t"     // r = m - x, m = (t0, a1)
        "subc.cc.u32 %1, a1, x1;\n\t"
        "subc.u32    m, 0, 0;\n\t"        // m = -borrow
        "sub.cc.u32  %0, %0, m;\n\t"      // on a borrow: r - EPS = r + p (mod 2^64)
        "subc.u32    %1, %1, 0;\n\t"
        "}"
        : "=&r"(r0), "=&r"(r1) : "r"(t0), "r"(t1), "r"(t2), "r"(t3));
    return mk(r0, r1);
  }
  // x * s mod p, canonical, for any 64-bit x and a table constant sR = s R mod p (< p)
  __device__ __forceinline__ static uint64_t mulm(uint64_t x, uint64_t sR) {
    const uint64_t lo = x * sR, hi = __umul64hi(x, sR);
    return mont_reduce(lo32(lo), hi32(lo), lo32(hi), hi32(hi));
  }
  __device__ __forceinline__ static uint64_t canon(uint64_t x) { return x >= P ? x - P : x; }

  // Butterflies: every twiddle / scaling operand is a table constant in Montgomery form (mulm);
  // the leaves multiply two variables (mul, plain reduction).
  // forward a: inputs weak; t = s y canonical -> single corrections
  __device__ __forceinline__ void fwd_a(uint64_t& x, uint64_t& y, uint64_t s) const {
    const uint64_t t = mulm(y, s);
    const uint64_t X = x;
    x = add_c(X, t);
    y = sub_c(X, t);
  }
  // forward b: t = s x canonical; t + y single correction; t - y with weak y needs two
  __device__ __forceinline__ void fwd_b(uint64_t& x, uint64_t& y, uint64_t s) const {
    const uint64_t t = mulm(x, s);
    const uint64_t Y = y;
    x = add_c(Y, t);
    y = sub_w(t, Y);
  }
  // forward b of a NEGATING level (sign-tracking vector split, fcirc_kernels.cuh `leaves` / neg_mask
  // and DESIGN.md section 9): the second output is stored negated, y - t instead of t - y -- with a
  // weak y, t - y needs two borrow corrections (sub_w, 8 instructions) and y - t one (sub_c, 5).  The
  // split is linear, so everything computed from the lower child carries the factor -1; the leaf
  // products take the accumulated sign back (leaf_neg: the operands of the Montgomery reduction's
  // final subtraction swapped, no extra instruction).  Negating are all column levels and the
  // sub-problem levels whose sign is free at the leaves.  NEG_B marks the fields that do this.
  static constexpr bool NEG_B = true;
  __device__ __forceinline__ void fwd_bn(uint64_t& x, uint64_t& y, uint64_t s) const {
    const uint64_t t = mulm(x, s);
    const uint64_t Y = y;
    x = add_c(Y, t);
    y = sub_c(Y, t);
  }
  // inverse: inputs canonical (leaf products and inverse outputs are canonical); outputs canonical.
  // (add_c and mul use the predicated corrections, like the forward butterflies.)
  __device__ __forceinline__ void inv(uint64_t& u, uint64_t& v, uint64_t si) const {
    const uint64_t s = add_c(u, v);   // u + v < 2p: one correction, result weak
    const uint64_t d = sub_c(u, v);   // canonical
    u = mulm(s, si);
    v = d;
  }
  __device__ __forceinline__ void inv_last(uint64_t& u, uint64_t& v, uint64_t si_k, uint64_t k) const {
    const uint64_t s = add_c(u, v);
    const uint64_t d = sub_c(u, v);
    u = mulm(s, si_k);
    v = mulm(d, k);
  }
  // x mod p for any 64-bit x: x >= p only if x_hi == 2^32 - 1 and x_lo != 0, and then x - p = (x_lo - 1, 0)
  __device__ __forceinline__ static uint64_t canon_w(uint64_t x) {
    uint32_t r0, r1;
    asm("{\n\t.reg .pred p, q;\n\t"
        "mov.u32         %0, %2;\n\t"
        "mov.u32         %1, %3;\n\t"
        "setp.eq.u32     p, %3, 0xffffffff;\n\t"
        "setp.ne.and.u32 q, %2, 0, p;\n\t"
        "@q sub.u32      %0, %2, 1;\n\t"
        "@q mov.u32      %1, 0;\n\t"
        "}"
        : "=&r"(r0), "=&r"(r1) : "r"(lo32(x)), "r"(hi32(x)));
    return mk(r0, r1);
  }
  // leaves (var x var): both factors are weak, so one is canonicalised first (mulm's precondition:
  // one factor < p) and the Montgomery reduction yields a b R^-1; the plan's scaling constants
  // carry the compensating R (api.cu: last_si and K are uploaded times R^2).
  __device__ __forceinline__ uint64_t leaf(uint64_t a, uint64_t b) const { return mulm(canon_w(a), b); }
  // -(a b R^-1): the leaf at a position whose b side arrives negated (fwd_bn)
  __device__ __forceinline__ uint64_t leaf_neg(uint64_t a, uint64_t b) const {
    const uint64_t x = canon_w(a);
    const uint64_t lo = x * b, hi = __umul64hi(x, b);
    return mont_reduce_neg(lo32(lo), hi32(lo), lo32(hi), hi32(hi));
  }
  __device__ __forceinline__ uint64_t single(uint64_t a, uint64_t b, uint64_t k) const {
    return mulm(leaf(a, b), k);
  }
};

// ------------------------------------------------------------------------------------------
// The paper's own ring: Z/pZ[sqrt 3], p = 2^31 - 1.  u + v sqrt 3 is packed as u | v << 32
// with canonical components (< p).  (a + b sqrt 3)(c + d sqrt 3) = (ac + 3bd) + (ad + bc) sqrt 3;
// the four 31x31-bit products and the sums fit in 64 bits (< 2^64), each component is then folded
// with 2^31 == 1 (mod p) twice and canonicalised once.  Context only: it
// reproduces the paper's arithmetic setting, the BASELINE configurations use Z/p.
// ------------------------------------------------------------------------------------------
struct FieldM31x2 {
  using T = uint64_t;
  using Tw = uint64_t;
  static constexpr uint32_t P = 0x7FFFFFFFu;

  __device__ __forceinline__ static uint32_t lo(uint64_t x) { return (uint32_t)x; }
  __device__ __forceinline__ static uint32_t hi(uint64_t x) { return (uint32_t)(x >> 32); }
  __device__ __forceinline__ static uint64_t pk(uint32_t u, uint32_t v) { return ((uint64_t)v << 32) | u; }
  // x < 2^64 -> x mod p in [0, p)
  __device__ __forceinline__ static uint32_t red(uint64_t x) {
    x = (x & P) + (x >> 31);                 // < 2^31 + 2^33
    x = (x & P) + (x >> 31);                 // <= 2^31 + 3
    const uint32_t r = (uint32_t)x;
    return r >= P ? r - P : r;
  }
  __device__ __forceinline__ static uint32_t addp(uint32_t a, uint32_t b) {
    const uint32_t s = a + b;
    return s >= P ? s - P : s;
  }
  __device__ __forceinline__ static uint32_t subp(uint32_t a, uint32_t b) { return a >= b ? a - b : a + P - b; }
  __device__ __forceinline__ static uint64_t add(uint64_t x, uint64_t y) { return pk(addp(lo(x), lo(y)), addp(hi(x), hi(y))); }
  __device__ __forceinline__ static uint64_t sub(uint64_t x, uint64_t y) { return pk(subp(lo(x), lo(y)), subp(hi(x), hi(y))); }
  __device__ __forceinline__ static uint64_t mul(uint64_t x, uint64_t y) {
    const uint64_t a = lo(x), b = hi(x), c = lo(y), d = hi(y);
    return pk(red(a * c + 3 * (b * d)), red(a * d + b * c));
  }

  __device__ __forceinline__ void fwd_a(uint64_t& x, uint64_t& y, uint64_t s) const {
    const uint64_t t = mul(y, s);
    const uint64_t X = x;
    x = add(X, t);
    y = sub(X, t);
  }
  static constexpr bool NEG_B = false;   // see FieldGold::fwd_bn
  __device__ __forceinline__ void fwd_bn(uint64_t& x, uint64_t& y, uint64_t s) const { fwd_b(x, y, s); }
  __device__ __forceinline__ void fwd_b(uint64_t& x, uint64_t& y, uint64_t s) const {
    const uint64_t t = mul(x, s);
    const uint64_t Y = y;
    x = add(t, Y);
    y = sub(t, Y);
  }
  __device__ __forceinline__ void inv(uint64_t& u, uint64_t& v, uint64_t si) const {
    const uint64_t s = add(u, v), d = sub(u, v);
    u = mul(s, si);
    v = d;
  }
  __device__ __forceinline__ void inv_last(uint64_t& u, uint64_t& v, uint64_t si_k, uint64_t k) const {
    const uint64_t s = add(u, v), d = sub(u, v);
    u = mul(s, si_k);
    v = mul(d, k);
  }
  __device__ __forceinline__ uint64_t leaf(uint64_t a, uint64_t b) const { return mul(a, b); }
  __device__ __forceinline__ uint64_t single(uint64_t a, uint64_t b, uint64_t k) const { return mul(mul(a, b), k); }
};

}  // namespace fcirc

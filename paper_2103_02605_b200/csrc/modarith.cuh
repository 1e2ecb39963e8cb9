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
//      64x64 -> 128 with IMAD.WIDE chains, then the special reduction
//      2^64 == 2^32 - 1 (=: EPS), 2^96 == -1 (mod p); no division, no table.
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

// ------------------------------------------------------------------------------------------
// 32-bit NTT primes
// ------------------------------------------------------------------------------------------
struct TwU32 {
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
  // leaves: inputs in [0, 4p); returns a b R^-1 mod p in [0, 2p)
  __device__ __forceinline__ uint32_t leaf(uint32_t a, uint32_t b) const {
    a = red1(red2(a));
    b = red1(red2(b));
    uint32_t lo = a * b;
    uint32_t hi = __umulhi(a, b);
    uint32_t m = lo * pinv_neg;
    // (a b + m p) / 2^32: the low words cancel exactly (lo + m p == 0 mod 2^32); carry = (lo != 0)
    uint32_t mh = __umulhi(m, p);
    return hi + mh + (lo != 0u);
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

  // a + b mod p on weakly reduced inputs (any 64-bit values); result weakly reduced
  __device__ __forceinline__ static uint64_t add(uint64_t a, uint64_t b) {
    uint64_t s = a + b;
    uint64_t c = (s < a) ? EPS : 0ull;  // wrapped: + 2^64 == + EPS
    uint64_t t = s + c;
    uint64_t c2 = (t < s) ? EPS : 0ull;
    return t + c2;
  }
  // a - b mod p on weakly reduced inputs
  __device__ __forceinline__ static uint64_t sub(uint64_t a, uint64_t b) {
    uint64_t d = a - b;
    uint64_t c = (a < b) ? EPS : 0ull;  // borrowed: - 2^64 == - EPS
    uint64_t t = d - c;
    uint64_t c2 = (d < c) ? EPS : 0ull;
    return t - c2;
  }
  // 64 x 64 -> 128 -> mod p (weakly reduced)
  __device__ __forceinline__ static uint64_t mul(uint64_t a, uint64_t b) {
    uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
    uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
    uint32_t t0, t1, t2, t3;
    asm("{\n\t"
        "mul.lo.u32      %0, %4, %6;\n\t"
        "mul.hi.u32      %1, %4, %6;\n\t"
        "mad.lo.cc.u32   %1, %4, %7, %1;\n\t"
        "madc.hi.u32     %2, %4, %7, 0;\n\t"
        "mad.lo.cc.u32   %1, %5, %6, %1;\n\t"
        "madc.hi.cc.u32  %2, %5, %6, %2;\n\t"
        "madc.hi.u32     %3, %5, %7, 0;\n\t"
        "mad.lo.cc.u32   %2, %5, %7, %2;\n\t"
        "addc.u32        %3, %3, 0;\n\t"
        "}"
        : "=r"(t0), "=r"(t1), "=r"(t2), "=r"(t3)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    // t = t0 + t1 2^32 + t2 2^64 + t3 2^96 == (t1:t0) - t3 + t2 (2^32 - 1)   (mod p)
    uint64_t lo = ((uint64_t)t1 << 32) | t0;
    uint64_t r = lo - t3;
    if (lo < (uint64_t)t3) r -= EPS;      // borrow: cannot borrow again (r >= 2^64 - 2^32)
    uint64_t m = ((uint64_t)t2 << 32) - t2;  // t2 (2^32 - 1) < 2^64
    uint64_t s = r + m;
    if (s < m) s += EPS;                   // carry: s < m - 1 here, so s + EPS cannot wrap
    return s;
  }
  __device__ __forceinline__ static uint64_t canon(uint64_t x) { return x >= P ? x - P : x; }

  __device__ __forceinline__ void fwd_a(uint64_t& x, uint64_t& y, uint64_t s) const {
    uint64_t t = mul(y, s);
    uint64_t X = x;
    x = add(X, t);
    y = sub(X, t);
  }
  __device__ __forceinline__ void fwd_b(uint64_t& x, uint64_t& y, uint64_t s) const {
    uint64_t t = mul(x, s);
    uint64_t Y = y;
    x = add(t, Y);
    y = sub(t, Y);
  }
  __device__ __forceinline__ void inv(uint64_t& u, uint64_t& v, uint64_t si) const {
    uint64_t s = add(u, v);
    uint64_t d = sub(u, v);
    u = mul(s, si);
    v = d;
  }
  __device__ __forceinline__ void inv_last(uint64_t& u, uint64_t& v, uint64_t si_k, uint64_t k) const {
    uint64_t s = add(u, v);
    uint64_t d = sub(u, v);
    u = canon(mul(s, si_k));
    v = canon(mul(d, k));
  }
  __device__ __forceinline__ uint64_t leaf(uint64_t a, uint64_t b) const { return mul(a, b); }
  __device__ __forceinline__ uint64_t single(uint64_t a, uint64_t b, uint64_t k) const {
    return canon(mul(mul(a, b), k));
  }
};

}  // namespace fcirc

// apps.cuh — kernels of the applications built on the f-circulant product.
//
// The polynomial embedding (row a~, zero padding, truncation) and the big-integer limb
// split are fused into the first / last pass of the product itself (fcirc_kernels.cuh EmbedIO).
// What remains here is the tail of the big-integer product (reading R12):
// Garner CRT of the three residues fused with the 16-bit digit sums and the per-segment carry
// summary (k_crt_digits), then the carry propagation (k_carry_top, k_carry_apply).
#pragma once
#include <cstdint>

#include "modarith.cuh"

namespace fcirc {

struct GarnerConsts {
  uint32_t p1, p2, p3;
  uint64_t p1p2;             // p1 p2 (< 2^59)
  uint32_t one2q, one3q;     // floor(2^32 / p2), floor(2^32 / p3): reduce a 32-bit value (Shoup, w = 1)
  uint32_t c12, c12q;        // p1^-1 mod p2 (Shoup pair)
  uint32_t p1m3, p1m3q;      // p1 mod p3
  uint32_t c123, c123q;      // (p1 p2)^-1 mod p3
};

// x w mod p for x < 2^32, with the Shoup quotient wq = floor(w 2^32 / p); canonical result
__device__ __forceinline__ uint32_t shoup_red(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
  const uint32_t r = x * w - __umulhi(x, wq) * p;   // in [0, 2p)
  return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }
__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t s = a + b;
  return s >= p ? s - p : s;
}

// V_k = CRT(r1, r2, r3) for one coefficient (Garner, mixed radix p1, p1 p2):
//   v1 = r1,  v2 = (r2 - v1) p1^-1 mod p2,  v3 = (r3 - v1 - v2 p1) (p1 p2)^-1 mod p3,
//   V = v1 + v2 p1 + v3 p1 p2 < p1 p2 p3 < 2^85, returned as (low 64 bits, high bits).
// (Within bigint_mul's size limit every coefficient is < 2^54 < p1 p2, so v3 = 0; the general
// three-prime reconstruction is kept as BASELINE.json's C5 route prescribes.)
__device__ __forceinline__ void garner(uint32_t r1, uint32_t r2, uint32_t r3, const GarnerConsts& g, uint64_t& lo,
                                       uint64_t& hi) {
  const uint32_t v1 = r1;
  const uint32_t v2 = shoup_red(sub_mod(r2, shoup_red(v1, 1u, g.one2q, g.p2), g.p2), g.c12, g.c12q, g.p2);
  const uint32_t t = add_mod(shoup_red(v1, 1u, g.one3q, g.p3), shoup_red(v2, g.p1m3, g.p1m3q, g.p3), g.p3);
  const uint32_t v3 = shoup_red(sub_mod(r3, t, g.p3), g.c123, g.c123q, g.p3);
  const unsigned __int128 val = (unsigned __int128)v1 + (unsigned __int128)v2 * g.p1 +
                                (unsigned __int128)v3 * g.p1p2;
  lo = (uint64_t)val;
  hi = (uint64_t)(val >> 64);
}

// ------------------------------------------------------------------------------------------
// carry propagation: E_j = e_j + g_j 2^16 with g_j in {0, 1}; digit j absorbs the carry c_j,
// c_{j+1} = g_j | (p_j & c_j), p_j = (e_j == 0xFFFF).  (G, P) pairs compose associatively
// (earlier segment X, later Y): (G_Y | (P_Y & G_X), P_Y & P_X).  Three launches:
//   k_crt_digits  per (integer, segment of kCarrySeg digits): CRT, digits and the segment's (G, P)
//   k_carry_top   per integer: exclusive scan over its segments -> carry into each segment
//   k_carry_apply per (integer, segment): block scan with the carry-in, write 32-bit words
// Each thread owns kCarryPer consecutive digits (coalesced uint4 loads).
// ------------------------------------------------------------------------------------------
constexpr int kCarryThreads = 256;
constexpr int kCarryPer = 8;
constexpr int kCarrySeg = kCarryThreads * kCarryPer;   // 2048 digits = 1024 output words

struct GP { uint32_t g, p; };
__device__ __forceinline__ GP gp_compose(GP x, GP y) { return {y.g | (y.p & x.g), y.p & x.p}; }  // x then y

// block-wide exclusive scan of (G, P) over NT threads (identity (0, 1)); returns this thread's
// prefix, *total
template <int NT = kCarryThreads>
__device__ __forceinline__ GP gp_block_exscan(GP v, GP* total) {
  __shared__ uint32_t wg[NT / 32], wp[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  GP inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    GP o{__shfl_up_sync(0xffffffffu, inc.g, off), __shfl_up_sync(0xffffffffu, inc.p, off)};
    if (lane >= off) inc = gp_compose(o, inc);
  }
  if (lane == 31) { wg[warp] = inc.g; wp[warp] = inc.p; }
  __syncthreads();
  GP wpre{0u, 1u};
  for (int w = 0; w < warp; ++w) wpre = gp_compose(wpre, GP{wg[w], wp[w]});
  GP tot{0u, 1u};
  for (int w = 0; w < NT / 32; ++w) tot = gp_compose(tot, GP{wg[w], wp[w]});
  *total = tot;
  GP ex{__shfl_up_sync(0xffffffffu, inc.g, 1), __shfl_up_sync(0xffffffffu, inc.p, 1)};
  if (lane == 0) ex = GP{0u, 1u};
  return gp_compose(wpre, ex);
}

__device__ __forceinline__ void load_digits(const uint32_t* Ei, int64_t nd, int64_t j0, uint32_t e[kCarryPer]) {
  if ((nd & 3) == 0 && j0 + kCarryPer <= nd) {   // 16-byte loads (E rows are 16-byte aligned)
    const uint4 x = reinterpret_cast<const uint4*>(Ei + j0)[0], y = reinterpret_cast<const uint4*>(Ei + j0)[1];
    e[0] = x.x; e[1] = x.y; e[2] = x.z; e[3] = x.w; e[4] = y.x; e[5] = y.y; e[6] = y.z; e[7] = y.w;
    return;
  }
#pragma unroll
  for (int q = 0; q < kCarryPer; ++q) e[q] = (j0 + q < nd) ? Ei[j0 + q] : 0u;
}

__device__ __forceinline__ GP local_gp(const uint32_t e[kCarryPer]) {
  GP acc{0u, 1u};
#pragma unroll
  for (int q = 0; q < kCarryPer; ++q) acc = gp_compose(acc, GP{e[q] >> 16, (e[q] & 0xFFFFu) == 0xFFFFu});
  return acc;
}

// One CTA per (integer, segment of kCarrySeg digits); thread t owns the kCarryPer digits
// j0 .. j0 + kCarryPer - 1, j0 = segment start + t kCarryPer.  The digit sums
//   D_j = sum_{i<6} chunk16_i(V_{j-i}) (< 6 * 2^16),  E_j = (D_j mod 2^16) + floor(D_{j-1} / 2^16)
// (< 2^16 + 6, so every carry is 0 or 1) need the CRT values V_k for k in [j0 - 6, j0 + 8): the
// thread computes its own 8 Garner reconstructions and takes the 6 below from its neighbour, all
// in registers -- no shared-memory chunk table (the former one ran into MIO throttling: 16.5
// stall cycles per issue, profiles/r01l_ncu_c5.txt).  It writes E for the final pass and the
// segment's carry-lookahead pair (G, P).
constexpr int kHalo = 6;
__global__ void __launch_bounds__(kCarryThreads)
k_crt_digits(const uint32_t* __restrict__ r1, const uint32_t* __restrict__ r2, const uint32_t* __restrict__ r3,
             int64_t L, int64_t ncoef, int64_t nd, int64_t nseg, GarnerConsts g, uint32_t* __restrict__ E,
             uint32_t* __restrict__ seg_gp) {
  pdl_entry();
  constexpr int NV = kCarryPer + kHalo;   // V_{j0 - kHalo + q}, q < NV
  const int64_t inst = blockIdx.x / nseg, sg = blockIdx.x - inst * nseg;
  const int64_t j0 = sg * kCarrySeg + (int64_t)threadIdx.x * kCarryPer;
  const uint32_t *a1 = r1 + inst * L, *a2 = r2 + inst * L, *a3 = r3 + inst * L;
  uint32_t w[NV][3];   // 96-bit V as three 32-bit words (V < p1 p2 p3 < 2^90)
  auto crt = [&](int q) {
    const int64_t k = j0 - kHalo + q;
    uint64_t lo = 0, hi = 0;
    if (k >= 0 && k < ncoef) garner(__ldg(a1 + k), __ldg(a2 + k), __ldg(a3 + k), g, lo, hi);
    w[q][0] = (uint32_t)lo;
    w[q][1] = (uint32_t)(lo >> 32);
    w[q][2] = (uint32_t)hi;
  };
  {   // this thread's own coefficients: 8 consecutive words per prime as two 16-byte loads when
      // they lie inside the instance's L-word residue arrays (j0 is a multiple of 8; the arrays are
      // 16-byte aligned for L % 4 == 0), else guarded scalar loads
    uint32_t v1[kCarryPer], v2[kCarryPer], v3[kCarryPer];
    if ((L & 3) != 0 || j0 + kCarryPer > L) {
#pragma unroll
      for (int d = 0; d < kCarryPer; ++d) {
        const bool in = j0 + d < ncoef;
        v1[d] = in ? __ldg(a1 + j0 + d) : 0u;
        v2[d] = in ? __ldg(a2 + j0 + d) : 0u;
        v3[d] = in ? __ldg(a3 + j0 + d) : 0u;
      }
    } else {
#pragma unroll
    for (int h = 0; h < kCarryPer; h += 4) {
      const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(a1 + j0 + h));
      const uint4 x2 = __ldg(reinterpret_cast<const uint4*>(a2 + j0 + h));
      const uint4 x3 = __ldg(reinterpret_cast<const uint4*>(a3 + j0 + h));
      v1[h] = x1.x; v1[h + 1] = x1.y; v1[h + 2] = x1.z; v1[h + 3] = x1.w;
      v2[h] = x2.x; v2[h + 1] = x2.y; v2[h + 2] = x2.z; v2[h + 3] = x2.w;
      v3[h] = x3.x; v3[h + 1] = x3.y; v3[h + 2] = x3.z; v3[h + 3] = x3.w;
    }
    }
#pragma unroll
    for (int d = 0; d < kCarryPer; ++d) {
      uint64_t lo = 0, hi = 0;
      if (j0 + d < ncoef) garner(v1[d], v2[d], v3[d], g, lo, hi);
      w[kHalo + d][0] = (uint32_t)lo;
      w[kHalo + d][1] = (uint32_t)(lo >> 32);
      w[kHalo + d][2] = (uint32_t)hi;
    }
  }
  // the halo rows 0..5 are the previous thread's last six: a warp shuffle, through shared memory
  // across warp boundaries, recomputed only by thread 0 (the previous segment's coefficients)
  __shared__ uint32_t edge[kCarryThreads / 32][kHalo][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 31)
#pragma unroll
    for (int r = 0; r < kHalo; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) edge[warp][r][c] = w[kCarryPer + r][c];
#pragma unroll
  for (int r = 0; r < kHalo; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) w[r][c] = __shfl_up_sync(0xffffffffu, w[kCarryPer + r][c], 1);
  __syncthreads();
  if (lane == 0) {
    if (warp > 0) {
#pragma unroll
      for (int r = 0; r < kHalo; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) w[r][c] = edge[warp - 1][r][c];
    } else {
#pragma unroll
      for (int q = 0; q < kHalo; ++q) crt(q);
    }
  }
  // 16-bit chunk i of V at row q
  auto chunk = [&](int q, int i) -> uint32_t { return (w[q][i >> 1] >> (16 * (i & 1))) & 0xFFFFu; };
  uint32_t e[kCarryPer];
#pragma unroll
  for (int d = 0; d < kCarryPer; ++d) {   // digit j = j0 + d uses rows d + kHalo - i
    uint32_t D = 0, Dm = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      D += chunk(d + kHalo - i, i);
      Dm += chunk(d + kHalo - 1 - i, i);
    }
    e[d] = (j0 + d < nd) ? (D & 0xFFFFu) + (Dm >> 16) : 0u;
  }
  uint32_t* Ei = E + inst * nd;
  if ((nd & 3) == 0 && j0 + kCarryPer <= nd) {   // 16-byte stores (E is our aligned workspace)
    reinterpret_cast<uint4*>(Ei + j0)[0] = make_uint4(e[0], e[1], e[2], e[3]);
    reinterpret_cast<uint4*>(Ei + j0)[1] = make_uint4(e[4], e[5], e[6], e[7]);
  } else {
#pragma unroll
    for (int d = 0; d < kCarryPer; ++d)
      if (j0 + d < nd) Ei[j0 + d] = e[d];
  }
  GP tot;
  gp_block_exscan(local_gp(e), &tot);
  if (threadIdx.x == 0) seg_gp[blockIdx.x] = tot.g | (tot.p << 1);
}

// one CTA of kTopThreads per integer: carry into every segment (exclusive scan of the segment
// pairs).  Each thread owns a contiguous run of segments, so all loads are independent (the former
// one-warp loop serialised a global-load round trip per 32 segments).
constexpr int kTopThreads = 1024;
__global__ void __launch_bounds__(kTopThreads) k_carry_top(uint32_t* __restrict__ seg_gp, int64_t nseg) {
  pdl_entry();
  uint32_t* s = seg_gp + (int64_t)blockIdx.x * nseg;
  const int64_t per = (nseg + kTopThreads - 1) / kTopThreads;
  const int64_t b0 = (int64_t)threadIdx.x * per, b1 = b0 + per < nseg ? b0 + per : nseg;
  GP agg{0u, 1u};
  for (int64_t i = b0; i < b1; ++i) agg = gp_compose(agg, GP{s[i] & 1u, s[i] >> 1});
  GP tot;
  GP c = gp_block_exscan<kTopThreads>(agg, &tot);   // carry-in state of segment b0 (g = carry)
  __syncthreads();                                   // every thread has read its run
  for (int64_t i = b0; i < b1; ++i) {
    const GP v{s[i] & 1u, s[i] >> 1};   // re-read (own run only: no other thread writes it)
    s[i] = c.g;                         // carry into segment i
    c = gp_compose(c, v);
  }
}

__global__ void __launch_bounds__(kCarryThreads)
k_carry_apply(const uint32_t* __restrict__ E, int64_t nd, int64_t nseg, const uint32_t* __restrict__ seg_cin,
              uint32_t* __restrict__ z, int64_t nw) {
  pdl_entry();
  const int64_t inst = blockIdx.x / nseg, sg = blockIdx.x - inst * nseg;
  const int64_t j0 = sg * kCarrySeg + (int64_t)threadIdx.x * kCarryPer;
  uint32_t e[kCarryPer];
  load_digits(E + inst * nd, nd, j0, e);
  GP tot;
  const GP pre = gp_block_exscan(local_gp(e), &tot);
  uint32_t c = pre.g | (pre.p & seg_cin[blockIdx.x]);   // carry into this thread's first digit
  uint32_t* zi = z + inst * nw;
  uint32_t out[kCarryPer / 2];
#pragma unroll
  for (int q = 0; q < kCarryPer; q += 2) {
    const uint32_t s0 = (e[q] & 0xFFFFu) + c;
    c = (e[q] >> 16) | (s0 >> 16);
    const uint32_t s1 = (e[q + 1] & 0xFFFFu) + c;
    c = (e[q + 1] >> 16) | (s1 >> 16);
    out[q >> 1] = (s0 & 0xFFFFu) | ((s1 & 0xFFFFu) << 16);
  }
  const int64_t w0 = j0 >> 1;   // kCarryPer / 2 = 4 output words
  if (w0 + 4 <= nw && (reinterpret_cast<uintptr_t>(zi + w0) & 15u) == 0) {
    *reinterpret_cast<uint4*>(zi + w0) = make_uint4(out[0], out[1], out[2], out[3]);
  } else {
#pragma unroll
    for (int q = 0; q < kCarryPer / 2; ++q)
      if (w0 + q < nw) zi[w0 + q] = out[q];
  }
}

}  // namespace fcirc

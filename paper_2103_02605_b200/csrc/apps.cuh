// apps.cuh — kernels of the applications built on the f-circulant product.
//
//   k_embed / k_truncate  polynomial product as an f = 1 circulant: the row is the
//                         index-reversed, zero-padded a~ (a~[0] = a[0], a~[L-m] = a[m]) so that
//                         (A(a~) b)_i = sum_j a[(i-j) mod L] b_j, the cyclic convolution, which
//                         equals the linear one because L >= na + nb - 1 (reading R8).
#pragma once
#include <cstdint>

namespace fcirc {

template <class E>
__global__ void k_embed(const E* __restrict__ a, int64_t na, const E* __restrict__ b, int64_t nb,
                        E* __restrict__ at, E* __restrict__ bp, int64_t L, int64_t batch) {
  const int64_t tot = batch * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = i / L, pos = i - inst * L;
    E va = 0;
    if (pos == 0) va = a[inst * na];
    else if (pos >= L - (na - 1)) va = a[inst * na + (L - pos)];
    at[i] = va;
    bp[i] = pos < nb ? b[inst * nb + pos] : (E)0;
  }
}

template <class E>
__global__ void k_truncate(const E* __restrict__ cf, int64_t L, E* __restrict__ c, int64_t nc, int64_t batch) {
  const int64_t tot = batch * nc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = i / nc, k = i - inst * nc;
    c[i] = cf[inst * L + k];
  }
}

}  // namespace fcirc

// ------------------------------------------------------------------------------------------
// large integers, reading R12: 16-bit limbs, three f = 1 circulant
// products mod 998244353 / 469762049 / 167772161, Garner CRT, carry propagation.
// ------------------------------------------------------------------------------------------
namespace fcirc {

__device__ __forceinline__ uint32_t limb16(const uint32_t* w, int64_t m) {
  return (w[m >> 1] >> (16 * (m & 1))) & 0xFFFFu;
}

// at = limb-row of x in the a~ embedding, bp = zero-padded limbs of y (limbs < 2^16 < every p)
__global__ void k_bigint_embed(const uint32_t* __restrict__ x, int64_t nx, const uint32_t* __restrict__ y,
                               int64_t ny, uint32_t* __restrict__ at, uint32_t* __restrict__ bp, int64_t L,
                               int64_t batch) {
  const int64_t tot = batch * L, lx = 2 * nx, ly = 2 * ny;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = i / L, pos = i - inst * L;
    const uint32_t* xi = x + inst * nx;
    uint32_t va = 0;
    if (pos == 0) va = limb16(xi, 0);
    else if (pos >= L - (lx - 1)) va = limb16(xi, L - pos);
    at[i] = va;
    bp[i] = pos < ly ? limb16(y + inst * ny, pos) : 0u;
  }
}

struct GarnerConsts {
  uint64_t p1, p2, p3;
  uint64_t inv_p1_mod_p2;      // p1^-1 mod p2
  uint64_t inv_p1p2_mod_p3;    // (p1 p2)^-1 mod p3
  uint64_t p1p2_mod_p3;
};

// V_k = CRT(r1, r2, r3) as a 128-bit integer (< p1 p2 p3 < 2^85), stored as two u64 words
__global__ void k_garner(const uint32_t* __restrict__ r1, const uint32_t* __restrict__ r2,
                         const uint32_t* __restrict__ r3, int64_t L, int64_t ncoef, int64_t batch, GarnerConsts g,
                         uint64_t* __restrict__ V) {
  const int64_t tot = batch * ncoef;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = i / ncoef, k = i - inst * ncoef;
    const uint64_t a1 = r1[inst * L + k], a2 = r2[inst * L + k], a3 = r3[inst * L + k];
    const uint64_t v1 = a1;
    const uint64_t v2 = ((a2 + g.p2 - (v1 % g.p2)) % g.p2) * g.inv_p1_mod_p2 % g.p2;
    // (a3 - v1 - v2 p1) mod p3
    const uint64_t t = (v1 % g.p3 + (v2 % g.p3) * (g.p1 % g.p3)) % g.p3;
    const uint64_t v3 = ((a3 + g.p3 - t) % g.p3) * g.inv_p1p2_mod_p3 % g.p3;
    const unsigned __int128 val = (unsigned __int128)v1 + (unsigned __int128)v2 * g.p1 +
                                  (unsigned __int128)v3 * ((unsigned __int128)g.p1 * g.p2);
    V[2 * i] = (uint64_t)val;
    V[2 * i + 1] = (uint64_t)(val >> 64);
  }
}

__device__ __forceinline__ uint32_t chunk16(const uint64_t* V, int64_t k, int i) {
  const uint64_t w = V[2 * k + (i >> 2)];
  return (uint32_t)(w >> (16 * (i & 3))) & 0xFFFFu;
}

// D_j = sum_{i<6} chunk_i(V_{j-i})  (< 6 * 2^16);  E_j = (D_j mod 2^16) + floor(D_{j-1} / 2^16)  (< 2^17)
__global__ void k_digits(const uint64_t* __restrict__ V, int64_t ncoef, int64_t nd, int64_t batch,
                         uint32_t* __restrict__ Eo) {
  const int64_t tot = batch * nd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = i / nd, j = i - inst * nd;
    const uint64_t* Vi = V + 2 * inst * ncoef;
    uint32_t D = 0, Dm = 0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (j - q >= 0 && j - q < ncoef) D += chunk16(Vi, j - q, q);
      if (j - 1 - q >= 0 && j - 1 - q < ncoef) Dm += chunk16(Vi, j - 1 - q, q);
    }
    Eo[i] = (D & 0xFFFFu) + (Dm >> 16);
  }
}

// carry-lookahead over E_j = e_j + g_j 2^16 (g_j in {0,1}): carry_out = g | (p & carry_in),
// p = (e == 0xFFFF).  One CTA per integer; thread-sequential chunks + block scan of (g, p).
constexpr int kCarryThreads = 1024;
__global__ void __launch_bounds__(kCarryThreads)
k_carry(const uint32_t* __restrict__ E, int64_t nd, uint32_t* __restrict__ z, int64_t nw, int* __restrict__ overflow) {
  const int64_t inst = blockIdx.x;
  const uint32_t* Ei = E + inst * nd;
  uint32_t* zi = z + inst * nw;
  const int64_t per = (nd + kCarryThreads - 1) / kCarryThreads;
  const int64_t j0 = threadIdx.x * per, j1 = min(nd, j0 + per);
  // local (g, p) of this chunk, composed left to right
  uint32_t G = 0, Pp = 1;
  for (int64_t j = j0; j < j1; ++j) {
    const uint32_t e = Ei[j];
    const uint32_t g = e >> 16, p = (e & 0xFFFFu) == 0xFFFFu;
    G = g | (p & G);
    Pp = Pp & p;
  }
  // exclusive scan across threads (carry into each chunk)
  __shared__ uint32_t sg[kCarryThreads], sp[kCarryThreads];
  sg[threadIdx.x] = G;
  sp[threadIdx.x] = Pp;
  __syncthreads();
  for (int off = 1; off < kCarryThreads; off <<= 1) {
    uint32_t g2 = 0, p2 = 1;
    if ((int)threadIdx.x >= off) { g2 = sg[threadIdx.x - off]; p2 = sp[threadIdx.x - off]; }
    __syncthreads();
    // (earlier block) then (this prefix): g = g_this | (p_this & g_earlier)
    const uint32_t gt = sg[threadIdx.x], pt = sp[threadIdx.x];
    sg[threadIdx.x] = gt | (pt & g2);
    sp[threadIdx.x] = pt & p2;
    __syncthreads();
  }
  uint32_t cin = threadIdx.x == 0 ? 0u : sg[threadIdx.x - 1];
  for (int64_t j = j0; j < j1; ++j) {
    const uint32_t e = Ei[j];
    const uint32_t s = (e & 0xFFFFu) + cin;
    const uint32_t d = s & 0xFFFFu;
    cin = (e >> 16) | (s >> 16);
    // digits j -> word j/2 (16-bit halves); each word is written by the thread owning its low digit
    if (j & 1) continue;
    uint32_t hi = 0;
    if (j + 1 < nd) {
      const uint32_t e1 = Ei[j + 1];
      hi = ((e1 & 0xFFFFu) + cin) & 0xFFFFu;
    }
    if ((j >> 1) < nw) zi[j >> 1] = d | (hi << 16);
  }
  if (overflow && threadIdx.x == kCarryThreads - 1 && cin) atomicExch(overflow, 1);
}

}  // namespace fcirc

// fcirc_kernels.cuh — sm_100a kernels of the f-circulant product.
//
// In-place iterative form of Algorithm 1 applied recursively.  The vector
// positions of one instance are addresses 0..n-1 (L = log2 n bits).  Level d (0 <= d < L) of the
// recursion pairs the addresses that differ in bit b = L-1-d; block e of level d holds the row of
// an f_{d,e}-circulant and uses the twiddle s_{d,e} = sqrt(f_{d,e}); its halves become the
// children 2e (f = +s) and 2e+1 (f = -s).  The twist table is heap-indexed: entry
// 2^d + e, which for an element at address x is (n + x) >> (b + 1).
//
// Kernels:
//   k_block   (K2 / K4) a sub-problem of size m = 2^M fully on chip: all its forward levels
//             for a and b (sharing each twiddle load), the leaves, all its inverse levels.
//             R elements per thread live in registers; each "phase" does r = log2 R levels in
//             registers, phases exchange through padded shared memory.  With k = 0 it is the
//             whole product (one HBM read of a and b, one write of c); with k > 0 it processes
//             the 2^k independent sub-products left after the top k levels (f_{k,E}-circulants).
//   k_cols    (K3 / K5) the top K levels, which act on columns (stride m = n / 2^K) of the
//             instance: forward for a and b (K3), or inverse incl. the global level 0 with the
//             1/n scaling and canonicalisation (K5).  Same register/shared-memory phase scheme
//             along the column; W consecutive columns per CTA for coalescing.
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "modarith.cuh"

namespace fcirc {

__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

// Phase geometry of a 2^NB-point transform done by threads holding R = 2^r points each.
// Phase 0 covers the top rp(0) = NB - r (NPH - 1) address bits (the short phase when r does not
// divide NB), every later phase r bits, the last one the lowest r.  Putting the short phase on top
// keeps every low phase a full r bits wide, which is what makes the smem swizzle below
// conflict-free in every phase (the top phase is contiguous across threads anyway).
template <int NB, int R>
struct Phases {
  static constexpr int r = ilog2c(R);
  static constexpr int T = (1 << NB) / R;            // threads per transform
  static constexpr int NPH = NB == 0 ? 0 : (NB + r - 1) / r;
  static __host__ __device__ constexpr int rp(int ph) { return ph == 0 ? NB - r * (NPH - 1) : r; }
  static __host__ __device__ constexpr int lo(int ph) { return NB - rp(0) - r * ph; }
  // runtime part of the address of thread t in phase ph (bits of t spread around the phase bits)
  static __device__ __forceinline__ int ins_t(int ph, int t) {
    const int l = lo(ph), w = rp(ph);
    return ((t >> l) << (l + w)) | (t & ((1 << l) - 1));
  }
  // compile-time part of the address of slot s in phase ph
  static __host__ __device__ constexpr int cslot(int ph, int s) {
    const int l = lo(ph), w = rp(ph);
    const int j = s & ((1 << w) - 1), g = s >> w;
    const int u = g * T;  // group offset in the thread-id space
    return ((u >> l) << (l + w)) | (j << l) | (u & ((1 << l) - 1));
  }
};

// Shared-memory swizzle of the phase exchanges: address x -> x ^ ((x >> r) & MASK), a GF(2)-linear
// bijection (so swz(a | b) = swz(a) ^ swz(b) for disjoint bit fields).  In a phase whose slot bits
// sit at [lo, lo + r), the thread bits above them are folded back onto the bank bits, so the 32
// threads of a warp (16 per wavefront for 8-byte elements) hit distinct banks in every phase
// (model: tools/bank_model.py; ncu: profiles/r01c_ncu_full_k_block_C4n20.txt had 25% conflicts
// with the former one-pad-per-16/32-elements layout).
template <class T> struct SwzMask;
template <> struct SwzMask<uint32_t> { static constexpr int V = 31; };  // 32 banks of 4 bytes
template <> struct SwzMask<uint64_t> { static constexpr int V = 15; };  // 16 8-byte lanes per wavefront

template <int R, class T>
__host__ __device__ __forceinline__ constexpr int swz(int x) {
  return x ^ ((x >> ilog2c(R)) & SwzMask<T>::V);
}

// ------------------------------------------------------------------------------------------
// Input/output modes of the first and last pass (embeddings fused into the loads,
// truncation into the stores, so the applications read no zero padding and write no scratch):
//   EMB_PLAIN   a, b, c are [batch][n] (fcirc_matvec)
//   EMB_POLY    polynomial product through an f = 1 circulant of order n (DESIGN.md
//               reading R8): row a~[0] = a[0], a~[pos] = a[n - pos] for pos > n - na, else 0;
//               vector b zero-padded; c truncated to nc = na + nb - 1 coefficients.
//   EMB_LIMBS   big integers: a, b are [batch][na | nb] little-endian 32-bit words read
//               as 16-bit limbs (row = reversed limbs of a, vector = limbs of b); c is [batch][n].
//   EMB_ANYN    Corollary 1: a circulant of any order na (= nb = nc) embedded in one of
//               order n (a power of two >= 2 na - 1): row a' = (a_0..a_{na-1}, 0..0, a_1..a_{na-1}),
//               vector b' = (b, 0..0); c = the first na entries of A' b'.
// ------------------------------------------------------------------------------------------
enum { EMB_PLAIN = 0, EMB_POLY = 1, EMB_LIMBS = 2, EMB_ANYN = 3 };
__host__ __device__ __forceinline__ bool emb_truncates(int mode) { return mode == EMB_POLY || mode == EMB_ANYN; }
struct EmbedIO {
  int mode = EMB_PLAIN;
  int64_t na = 0, nb = 0;   // EMB_POLY: coefficients per instance; EMB_LIMBS: 32-bit words
  int64_t nc = 0;           // EMB_POLY: output coefficients per instance
};

template <class T>
__device__ __forceinline__ T limb_at(const T* w, uint32_t m) {
  if constexpr (sizeof(T) == 4) return (__ldg(w + (m >> 1)) >> (16 * (m & 1))) & 0xFFFFu;
  else return 0;  // limbs are only used with the 32-bit primes
}
// Element `pos` (< n <= 2^24) of the row (SECOND = false) or the vector (SECOND = true) of caller
// instance `inst`, for the compile-time embedding MODE (the kernels are instantiated per mode: with a
// run-time mode switch every embedded load carried all four index paths in 64-bit arithmetic, 3x the
// SASS of the plain column pass).  Zero padding is never read.
template <int MODE, bool SECOND, class T>
__device__ __forceinline__ T io_load(const T* src, int64_t inst, uint32_t pos, uint32_t n, const EmbedIO& io) {
  if constexpr (MODE == EMB_PLAIN) {
    return src[inst * n + pos];
  } else if constexpr (MODE == EMB_POLY) {
    const uint32_t na = (uint32_t)io.na, nb = (uint32_t)io.nb;
    if constexpr (SECOND) return pos < nb ? src[inst * io.nb + pos] : (T)0;
    const T* ai = src + inst * io.na;
    return pos == 0 ? ai[0] : (pos > n - na ? ai[n - pos] : (T)0);
  } else if constexpr (MODE == EMB_ANYN) {
    const uint32_t na = (uint32_t)io.na, nb = (uint32_t)io.nb;
    if constexpr (SECOND) return pos < nb ? src[inst * io.nb + pos] : (T)0;
    const T* ai = src + inst * io.na;
    return pos < na ? ai[pos] : (pos > n - na ? ai[pos - (n - na)] : (T)0);
  } else {   // EMB_LIMBS: na, nb are 32-bit words (2 limbs each)
    const uint32_t la = 2 * (uint32_t)io.na, lb = 2 * (uint32_t)io.nb;
    if constexpr (SECOND) return pos < lb ? limb_at(src + inst * io.nb, pos) : (T)0;
    const T* xi = src + inst * io.na;
    return pos == 0 ? limb_at(xi, 0u) : (pos > n - la ? limb_at(xi, n - pos) : (T)0);
  }
}
template <int MODE, class T>
__device__ __forceinline__ void io_store(T* dst, int64_t inst, uint32_t pos, uint32_t n, T v, const EmbedIO& io) {
  if constexpr (MODE == EMB_POLY || MODE == EMB_ANYN) {
    if (pos < (uint32_t)io.nc) dst[inst * io.nc + pos] = v;
  } else {
    dst[inst * (int64_t)n + pos] = v;
  }
}

// ------------------------------------------------------------------------------------------
// Several 32-bit primes in ONE launch (bigint_mul's three CRT products):
// instance j of the launch belongs to prime q = (inst0 + j) / per and reads the operands of instance
// (inst0 + j) % per; each prime brings its field constants and twist tables.  A CTA that stages
// twiddles in shared memory serves one prime only (the launcher keeps its instance groups inside
// one prime); unstaged kernels select per thread.
// ------------------------------------------------------------------------------------------
struct PrimeSel {
  FieldU32 fld;
  const TwU32* twf;
  const TwU32* twi;
  TwU32 last_si, last_k;
};
struct MultiPrime {
  int n = 1;             // primes in the launch (the FieldU32M kernels read it; others ignore it)
  int64_t per = 1;       // instances per prime
  int64_t inst0 = 0;     // global instance index of the launch's instance 0 (multi-pass chunks)
  PrimeSel ps[3];
};
// the field constants and tables an instance uses
template <class F>
struct FieldView {
  F fld;
  const typename F::Tw* twf;
  const typename F::Tw* twi;
  typename F::Tw last_si, last_k;
};
// The multi-prime kernels are the FieldU32M instantiations, a distinct field type, so that the
// single-field kernels carry neither the prime table in their parameters nor the selection code:
// both measurably changed ptxas's output for the register-tight u32 column passes (a run-time
// branch: C3 -18 %; a larger parameter block or local copies of the parameters: +8..25 % SASS in
// the embedded u32 column passes, C3 -9 %; profiles/r02c_ab*.txt).
struct FieldU32M : FieldU32 {};
template <class F>
constexpr bool kMulti = std::is_same<F, FieldU32M>::value;

// Single-field kernels get an empty view and keep reading the kernel parameters at their uses.
struct NoView {};
template <class F, class A>
__device__ __forceinline__ auto field_view(const F& fld, const A& args, int64_t inst) {
  if constexpr (kMulti<F>) {
    const uint32_t q = (uint32_t)(args.mp.inst0 + inst) / (uint32_t)args.mp.per;   // < 2^31 instances
    const PrimeSel& ps = q == 0 ? args.mp.ps[0] : (q == 1 ? args.mp.ps[1] : args.mp.ps[2]);
    return FieldView<F>{F{ps.fld}, ps.twf, ps.twi, ps.last_si, ps.last_k};
  } else {
    (void)fld; (void)args; (void)inst;
    return NoView{};
  }
}
template <class F> __device__ __forceinline__ const F& select_field(const FieldView<F>& v, const F&) { return v.fld; }
template <class F> __device__ __forceinline__ const F& select_field(const NoView&, const F& param) { return param; }
template <class F, class A> __device__ __forceinline__ const typename F::Tw* view_twf(const FieldView<F>& v, const A&) { return v.twf; }
template <class F, class A> __device__ __forceinline__ const typename F::Tw* view_twf(const NoView&, const A& a) { return a.twf; }
template <class F, class A> __device__ __forceinline__ const typename F::Tw* view_twi(const FieldView<F>& v, const A&) { return v.twi; }
template <class F, class A> __device__ __forceinline__ const typename F::Tw* view_twi(const NoView&, const A& a) { return a.twi; }
template <class F, class A> __device__ __forceinline__ typename F::Tw view_lsi(const FieldView<F>& v, const A&) { return v.last_si; }
template <class F, class A> __device__ __forceinline__ typename F::Tw view_lsi(const NoView&, const A& a) { return a.last_si; }
template <class F, class A> __device__ __forceinline__ typename F::Tw view_lk(const FieldView<F>& v, const A&) { return v.last_k; }
template <class F, class A> __device__ __forceinline__ typename F::Tw view_lk(const NoView&, const A& a) { return a.last_k; }
// the caller's instance whose operands instance `inst` of the launch reads
template <class F, class A>
__device__ __forceinline__ int64_t src_inst(const A& args, int64_t inst) {
  if constexpr (kMulti<F>) return (uint32_t)(args.mp.inst0 + inst) % (uint32_t)args.mp.per;
  else return inst;
}

// ------------------------------------------------------------------------------------------
// Building blocks of the register/shared-memory phase scheme, shared by every kernel below.
//   exchange / exchange2  move the R register values of one (or two) arrays from the layout of
//                         phase ph_from to that of ph_to through shared memory; idx(base, slot)
//                         maps an address (k_block: position, k_cols: row) given as its thread
//                         part plus its compile-time slot part to the swizzled smem index
//   forward_phase         the split levels of phase ph, top address bit first: bf(s0, s1, bit, tb, cs)
//                         gets the two slots of a butterfly pair, the pair bit and the address
//                         tb | cs of slot s0 split into its thread part tb and its compile-time
//                         slot part cs (disjoint bits), so twiddle indices separate the same way
//   inverse_phase         the recombination levels of phase ph, low address bit first
// All loops are fully unrolled (compile-time slots), so the register arrays stay in registers.
// ------------------------------------------------------------------------------------------
// One barrier per exchange (read-after-write).  No barrier is needed between an exchange's reads
// and the next exchange's writes to the same buffer: a thread reads the addresses of the slots it
// holds in phase ph_to and the next exchange (from ph_to) writes exactly those addresses, so it
// only overwrites values it has already read itself.  Callers that reuse the buffer with another
// layout (k_cols_tma between tiles) synchronise themselves.
// barrier of an exchange: the whole CTA, or (k_block_pipe) one named barrier per independent
// thread group of a CTA
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct NamedSync {
  int id, nthreads;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  }
};

template <class PH, int R, class T, class Idx, class Sync = CtaSync>
__device__ __forceinline__ void exchange(T (&x)[R], T* buf, int ph_from, int ph_to, int t, Idx idx, Sync sync = Sync{}) {
  const int wb = PH::ins_t(ph_from, t);
#pragma unroll
  for (int s = 0; s < R; ++s) buf[idx(wb, PH::cslot(ph_from, s))] = x[s];
  sync();
  const int rb = PH::ins_t(ph_to, t);
#pragma unroll
  for (int s = 0; s < R; ++s) x[s] = buf[idx(rb, PH::cslot(ph_to, s))];
}

template <class PH, int R, class T, class Idx, class Sync = CtaSync>
__device__ __forceinline__ void exchange2(T (&x)[R], T (&y)[R], T* bx, T* by, int ph_from, int ph_to, int t, Idx idx,
                                          Sync sync = Sync{}) {
  const int wb = PH::ins_t(ph_from, t);
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int ad = idx(wb, PH::cslot(ph_from, s));
    bx[ad] = x[s];
    by[ad] = y[s];
  }
  sync();
  const int rb = PH::ins_t(ph_to, t);
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int ad = idx(rb, PH::cslot(ph_to, s));
    x[s] = bx[ad];
    y[s] = by[ad];
  }
}

// In-warp alternative to the LAST exchange (phases NPH-2 <-> NPH-1 of a 2^M-point transform with
// R = 2^r points per thread): there the exchanged address bits are the low r thread bits, i.e. lanes
// of one group of R consecutive lanes, and the exchange is an R x R transpose within each group:
// r butterfly stages of __shfl_xor_sync (stage k swaps the slots whose bit k differs from the lane's
// bit k with lane ^ 2^k), no shared memory and no barrier.  (North-star mechanism "warp-shuffle
// exchanges for the innermost levels"; measured against the shared-memory exchange.)
template <int R, class T>
__device__ __forceinline__ void lane_transpose(T (&x)[R], int lane) {
#pragma unroll
  for (int k = 0; (1 << k) < R; ++k) {
    const int b = 1 << k;
    const bool upper = (lane >> k) & 1;
#pragma unroll
    for (int s0 = 0; s0 < R; ++s0) {
      if (s0 & b) continue;
      const T send = upper ? x[s0] : x[s0 | b];
      const T recv = __shfl_xor_sync(0xffffffffu, send, b);
      if (upper) x[s0] = recv;
      else x[s0 | b] = recv;
    }
  }
}

template <class PH, int R, class BF>
__device__ __forceinline__ void forward_phase(int ph, int t, BF bf) {
  const int rp = PH::rp(ph), lo = PH::lo(ph), tins = PH::ins_t(ph, t);
#pragma unroll
  for (int l = 0; l < rp; ++l) {
    const int jb = rp - 1 - l;
#pragma unroll
    for (int s0 = 0; s0 < R; ++s0) {
      if ((s0 >> jb) & 1) continue;
      bf(s0, s0 + (1 << jb), lo + jb, tins, PH::cslot(ph, s0));
    }
  }
}

template <class PH, int R, class BF>
__device__ __forceinline__ void inverse_phase(int ph, int t, BF bf) {
  const int rp = PH::rp(ph), lo = PH::lo(ph), tins = PH::ins_t(ph, t);
#pragma unroll
  for (int jb = 0; jb < rp; ++jb) {
#pragma unroll
    for (int s0 = 0; s0 < R; ++s0) {
      if ((s0 >> jb) & 1) continue;
      bf(s0, s0 + (1 << jb), lo + jb, tins, PH::cslot(ph, s0));
    }
  }
}

// Sign-tracking vector split (fields with F::NEG_B, FieldGold).  The b butterfly's second output
// s x - y is a canonical-minus-weak subtraction (two borrow corrections); its negative y - s x needs
// one (fwd_bn).  A level that stores the negative multiplies, by linearity, everything below the
// lower child by -1, so the b leaf at address x of sub-block E arrives times
// (-1)^(popcount(E) + popcount(x & NEGMASK)), NEGMASK the address bits of the negating levels of the
// sub-problem (all K column levels negate: popcount(E)).  The leaf product takes that sign back
// (leaf_neg: the operands of the Montgomery reduction's final subtraction swapped, same instruction
// count).  Negating are the levels whose sign costs nothing at the leaves, where address = t << r | slot:
//   * bits [0, r): slot bits -- the sign is a compile-time property of the slot;
//   * bits >= r + 5: thread bits >= 5 -- the sign is uniform over a warp (with E: one non-divergent branch);
// the five levels in between (lane bits) keep the plain butterfly (their sign would differ per lane:
// the conditional negations cost what those levels save, profiles/r02t_ab_negb_hyb_pred.txt).
template <class PH>
__host__ __device__ constexpr int neg_mask() {
  constexpr int RL = PH::rp(PH::NPH - 1);
  return ((1 << RL) - 1) | ~((1 << (RL + 5)) - 1);
}
template <class PH, class F>
__host__ __device__ constexpr bool neg_level(int bit) {
  if constexpr (F::NEG_B) return (neg_mask<PH>() >> bit) & 1;
  else return false;
}
template <class PH, class F, int R, class T>
__device__ __forceinline__ void leaves(const F& fld, T (&xm)[R], const T (&xa)[R], const T (&xb)[R], int E, int t) {
  if constexpr (F::NEG_B) {
    constexpr int L = PH::NPH - 1;
    static_assert(PH::lo(L) == 0, "leaf layout: address = t << r | slot");
    if ((__popc(E) + __popc(t >> 5)) & 1) {   // warp-uniform
#pragma unroll
      for (int s = 0; s < R; ++s)
        xm[s] = (__builtin_popcount(PH::cslot(L, s) & neg_mask<PH>()) & 1) ? fld.leaf(xa[s], xb[s]) : fld.leaf_neg(xa[s], xb[s]);
    } else {
#pragma unroll
      for (int s = 0; s < R; ++s)
        xm[s] = (__builtin_popcount(PH::cslot(L, s) & neg_mask<PH>()) & 1) ? fld.leaf_neg(xa[s], xb[s]) : fld.leaf(xa[s], xb[s]);
    }
  } else {
    (void)E; (void)t;
#pragma unroll
    for (int s = 0; s < R; ++s) xm[s] = fld.leaf(xa[s], xb[s]);
  }
}

// Instance base pointer as an opaque value: element accesses p[off] with a 32-bit row offset then
// compile to one IMAD.WIDE.U32 (off * sizeof(T) + p) instead of a re-associated 64-bit index
// computation (shift, add, add-with-carry).  Used where it measured faster: the Goldilocks forward
// column pass (-3 %; the u32 column passes and the TMA inverse measured 2-9 % slower with it,
// profiles/r01i_sweep_col_offsets_ab.txt).
template <class P>
__device__ __forceinline__ P* opaque(P* p) {
  asm("" : "+l"(p));
  return p;
}

// read-only twiddle load through the non-coherent (texture) path: the tables are immutable for the
// lifetime of a plan, and the top levels of every phase are shared by many threads of a CTA
__device__ __forceinline__ uint64_t ldtw(const uint64_t* p) { return __ldg(p); }
__device__ __forceinline__ TwU32 ldtw(const TwU32* p) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  return TwU32{v.x, v.y};
}

// ------------------------------------------------------------------------------------------
// k_block: fused sub-problem kernel
// ------------------------------------------------------------------------------------------
template <class F>
struct BlockArgs {
  const typename F::T* a;   // a' (row, after the top k levels), [units][m]
  const typename F::T* b;   // b'
  typename F::T* out;       // M (k > 0) or c (k == 0); may alias a
  int64_t units;            // batch * 2^k
  int k;                    // levels above this kernel (0: whole problem); grid = 2^k x
                            // ceil(batch / IPC), CTA b: sub-block E = b mod 2^k, instances (b >> k) IPC + li
  const typename F::Tw* twf;  // heap-indexed s_{d,e}
  const typename F::Tw* twi;  // heap-indexed s_{d,e}^-1
  typename F::Tw last_si;   // s_{0,0}^-1 * K   (used when k == 0)
  typename F::Tw last_k;    // K = n^-1 (x R for FieldU32)
  EmbedIO io;               // k == 0 and EMB only: embedding of the loads / truncation of the stores
  int seq = 1;              // instance groups per CTA, one after another (sharing staged twiddles)
};
// kernel argument type (see ColKArgs below): the multi-prime instantiations add the prime table
template <class F> struct BlockArgsM : BlockArgs<F> { MultiPrime mp; };
template <class F> using BlockKArgs = typename std::conditional<kMulti<F>, BlockArgsM<F>, BlockArgs<F>>::type;

// k_block stages its twiddle slices in shared memory for the 32-bit fields (see TWS below), at
// swizzled positions i ^ ((i >> 4) & 31) (a bijection of [0, 2^M)): the model in
// tools/bank_model.py gives 1.2x the conflict-free wavefronts instead of 1.5x unswizzled
__device__ __forceinline__ int tw_swz(int i) { return i ^ ((i >> 4) & 31); }
template <class F, int M> struct TwStage { static constexpr bool value = false; };
template <int M> struct TwStage<FieldU32, M> { static constexpr bool value = M >= 6; };
template <int M> struct TwStage<FieldU32M, M> { static constexpr bool value = M >= 6; };

template <class F, int M, int R, int IPC, int MINB = 1, int EMB = EMB_PLAIN, bool TWS = false, bool SHF = false>
__global__ void __launch_bounds__((1 << M) / R * IPC, MINB)
k_block(F fld0, BlockKArgs<F> args) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<M, R>;
  constexpr int m = 1 << M;
  constexpr int TT = PH::T;
  constexpr int NPH = PH::NPH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);

  const int t = threadIdx.x % TT;
  const int li = threadIdx.x / TT;
  T* sa = sm + (size_t)li * 2 * m;   // swizzled, unpadded
  T* sb = sa + m;
  // swz is GF(2)-linear: swz(base | slot) = swz(base) ^ swz(slot), the latter a compile-time constant
  auto idx = [](int base_part, int slot_part) { return swz<R, T>(base_part) ^ swz<R, T>(slot_part); };

  const int k = args.k;
  const int64_t batch = args.units >> k;
  const int nseq = TWS ? args.seq : 1;   // unstaged launches: one group (no loop, no extra registers)
  // field and tables: per CTA when staged (the launcher keeps a staged CTA inside one prime), else
  // per instance group (the only group of the thread)
  const auto fv = field_view(fld0, args, ((int64_t)(blockIdx.x >> k) * nseq) * IPC + (TWS ? 0 : li));
  const F& fld = select_field(fv, fld0);

  // Twiddle staging (32-bit fields): sub-block E uses the heap slice
  // {2^(k+j) + E 2^j + e' : j < M, e' < 2^j} of each table (contiguous per level).
  // It is copied, coalesced, into shared memory at local heap index 2^j + e' (1-based), so the
  // butterflies read twiddles with LDS instead of scattered L2 loads (profiles/r01c: the u32
  // k_block stalled on long_scoreboard).  Goldilocks is arithmetic-bound and keeps the LDG path;
  // so does the fused whole-product launch (k = 0), whose CTAs all share one table via L1/L2.
  Tw* twsf = reinterpret_cast<Tw*>(sm + (size_t)IPC * 2 * m);
  Tw* twsi = twsf + m;
  auto stage = [&](int E) {
    for (int h = threadIdx.x + 1; h < m; h += blockDim.x) {
      const int j = 31 - __clz(h);
      const int g = (1 << (k + j)) + (E << j) + (h - (1 << j));
      twsf[tw_swz(h)] = view_twf<F>(fv, args)[g];
      twsi[tw_swz(h)] = view_twi<F>(fv, args)[g];
    }
  };
  int gbase = 0;   // heap-extended address base of the current sub-block (fits: < 2n <= 2^24)
  // twiddle of the pair bit `bit` at address x = tb | cs: heap entry (gbase | x) >> (bit+1), whose
  // thread part (gbase | tb) >> (bit+1) is shared by every slot of a level and whose slot part
  // cs >> (bit+1) is a compile-time offset (disjoint bits: the sum is the OR).  Staged: local heap
  // index 2^(M-1-bit) | (x >> (bit+1)), swizzled with the GF(2)-linear tw_swz term by term.
  auto tw_at = [&](const Tw* table, const Tw* staged, int bit, int tb, int cs) -> Tw {
    if constexpr (TWS) return staged[tw_swz(1 << (M - 1 - bit)) ^ tw_swz(tb >> (bit + 1)) ^ tw_swz(cs >> (bit + 1))];
    else return ldtw(table + ((gbase | tb) >> (bit + 1)) + (cs >> (bit + 1)));
  };

  // Work assignment: CTA b -> sub-block E = b mod 2^k and seq consecutive instance groups
  // (b >> k) seq + it, it < seq, of IPC instances each.  seq > 1 (staged launches) stages the
  // twiddle slice once per seq sub-problems (S1 k_block -14 %).  No
  // barrier between them: the next one's first exchange writes sa at the addresses this thread
  // read last (exchange rule) and sb, last read in the forward levels, only after the inverse
  // exchanges' CTA barriers.
  const int E = (int)(blockIdx.x & ((1u << k) - 1));
  gbase = ((1 << k) + E) << M;
  if constexpr (TWS) {
    stage(E);
    __syncthreads();
  }
  for (int it = 0; it < nseq; ++it) {
  const int64_t inst = ((int64_t)(blockIdx.x >> k) * nseq + it) * IPC + li;
  const bool active = inst < batch;
  const int64_t base = ((inst << k) + E) * m;

  T xa[R], xb[R];
  // ---- load (phase-0 addresses: slot s at s * 2^lo + t, coalesced across t)
  if (active) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int ad = PH::ins_t(0, t) + PH::cslot(0, s);
      if constexpr (EMB) {
        xa[s] = io_load<EMB, false>(args.a, src_inst<F>(args, inst), ad, m, args.io);
        xb[s] = io_load<EMB, true>(args.b, src_inst<F>(args, inst), ad, m, args.io);
      } else {
        xa[s] = args.a[base + ad];
        xb[s] = args.b[base + ad];
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < R; ++s) xa[s] = xb[s] = 0;
  }

  // ---- forward levels (Algorithm 1 split of a and b, sharing each twiddle), phase by phase
  static_assert(!SHF || (NPH >= 2 && PH::rp(NPH - 2) == PH::r && PH::lo(NPH - 2) == PH::r),
                "lane_transpose needs full-width last two phases");
#pragma unroll
  for (int ph = 0; ph < NPH; ++ph) {
    if constexpr (SHF && NPH >= 2) {
      if (ph == NPH - 1) {
        lane_transpose<R>(xa, t & (R - 1));
        lane_transpose<R>(xb, t & (R - 1));
      } else if (ph > 0) {
        exchange2<PH, R>(xa, xb, sa, sb, ph - 1, ph, t, idx);
      }
    } else {
      if (ph > 0) exchange2<PH, R>(xa, xb, sa, sb, ph - 1, ph, t, idx);
    }
    forward_phase<PH, R>(ph, t, [&](int s0, int s1, int bit, int tb, int cs) {
      const Tw tw = tw_at(view_twf<F>(fv, args), twsf, bit, tb, cs);
      fld.fwd_a(xa[s0], xa[s1], tw);
      if (neg_level<PH, F>(bit)) fld.fwd_bn(xb[s0], xb[s1], tw);   // compile-time after unrolling
      else fld.fwd_b(xb[s0], xb[s1], tw);
    });
  }

  // ---- leaves: 1x1 products (the recursion bottom), same thread/slot layout
  if constexpr (M == 0) {
    if (active) {
      const T v = fld.single(xa[0], xb[0], view_lk<F>(fv, args));
      if constexpr (EMB) io_store<EMB>(args.out, inst, 0, 1, v, args.io);
      else args.out[base] = v;
    }
  } else {
    T xm[R];
    leaves<PH, F, R>(fld, xm, xa, xb, E, t);

    // ---- inverse levels (recombination c1 = (M1+M2)/(2s), c2 = (M1-M2)/2), low bits first
    const bool top = (k == 0);
#pragma unroll
    for (int ph = NPH - 1; ph >= 0; --ph) {
      if constexpr (SHF && NPH >= 2) {
        if (ph == NPH - 2) lane_transpose<R>(xm, t & (R - 1));
        else if (ph < NPH - 1) exchange<PH, R>(xm, sa, ph + 1, ph, t, idx);
      } else {
        if (ph < NPH - 1) exchange<PH, R>(xm, sa, ph + 1, ph, t, idx);
      }
      inverse_phase<PH, R>(ph, t, [&](int s0, int s1, int bit, int tb, int cs) {
        if (bit == M - 1 && top) fld.inv_last(xm[s0], xm[s1], view_lsi<F>(fv, args), view_lk<F>(fv, args));
        else fld.inv(xm[s0], xm[s1], tw_at(view_twi<F>(fv, args), twsi, bit, tb, cs));
      });
    }

    // ---- store (phase-0 addresses, coalesced)
    if (active) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int ad = PH::ins_t(0, t) + PH::cslot(0, s);
        if constexpr (EMB) io_store<EMB>(args.out, inst, ad, m, xm[s], args.io);
        else args.out[base + ad] = xm[s];
      }
    }
  }
  }   // instance groups of the CTA
}

// ------------------------------------------------------------------------------------------
// Column passes: the top K levels, along columns of stride m = n / 2^K
// ------------------------------------------------------------------------------------------
template <class F>
struct ColArgs {
  const typename F::T* src0;  // forward: a      inverse: M
  const typename F::T* src1;  // forward: b      inverse: unused
  typename F::T* dst0;        // forward: a'     inverse: c (may alias src0)
  typename F::T* dst1;        // forward: b'
  int64_t m;                  // column stride = n >> K
  int64_t n;
  int64_t colblocks;          // m / (W * column groups per thread)
  int64_t units;              // instances * colblocks
  const typename F::Tw* twf;
  const typename F::Tw* twi;
  typename F::Tw last_si;
  typename F::Tw last_k;
  EmbedIO io;                 // EMB only: forward embedding of the loads; inverse truncation of the stores
};

// Kernel argument types: the FieldU32M (multi-prime) instantiations take the argument struct plus
// the prime table; every other field takes the plain struct (unchanged parameter block).
template <class F> struct ColArgsM : ColArgs<F> { MultiPrime mp; };
template <class F> using ColKArgs = typename std::conditional<kMulti<F>, ColArgsM<F>, ColArgs<F>>::type;
// colblocks (= m / W or m / (2 W)) is a power of two: the block -> (instance, column block) split is a
// shift and a mask instead of a 64-bit division per thread
template <class A>
__device__ __forceinline__ int cb_log(const A& args) { return __ffsll((long long)args.colblocks) - 1; }

// row swizzle (GF(2)-linear bijection of [0, 2^K)): with the short phase on top, the rows a warp
// touches in one access land in distinct banks in every phase (tools/bank_model.py)
template <class PH, int W>
struct ColIdx {
  int c;
  __device__ __forceinline__ int operator()(int row) const { return (row ^ ((row >> PH::r) & 7)) * W + c; }
  __device__ __forceinline__ int operator()(int base_part, int slot_part) const { return (*this)(base_part + slot_part); }
};

// twiddles of the column levels: heap entry (2^K | row) >> (bit + 1), the same for every column;
// row = tb | cs (thread part, compile-time slot part; disjoint bits) as in k_block
template <int K, class Tw>
__device__ __forceinline__ Tw col_tw(const Tw* table, int bit, int tb, int cs) {
  return ldtw(table + (((1 << K) | tb) >> (bit + 1)) + (cs >> (bit + 1)));
}

// The K forward levels of NG register arrays (same rows), NG in {1, 2}: bf runs the butterflies.
template <class PH, int K, int R, int NPH, class T, class Idx, class BF>
__device__ __forceinline__ void col_forward(T (&x)[R], T (*y)[R], T* bx, T* by, int t, Idx idx, BF bf) {
#pragma unroll
  for (int ph = 0; ph < NPH; ++ph) {
    if (ph > 0) {
      if (y) exchange2<PH, R>(x, *y, bx, by, ph - 1, ph, t, idx);
      else exchange<PH, R>(x, bx, ph - 1, ph, t, idx);
    }
    forward_phase<PH, R>(ph, t, bf);
  }
}

template <class PH, int K, int R, int NPH, class T, class Idx, class BF>
__device__ __forceinline__ void col_inverse(T (&x)[R], T (*y)[R], T* bx, T* by, int t, Idx idx, BF bf) {
#pragma unroll
  for (int ph = NPH - 1; ph >= 0; --ph) {
    if (ph < NPH - 1) {
      if (y) exchange2<PH, R>(x, *y, bx, by, ph + 1, ph, t, idx);
      else exchange<PH, R>(x, bx, ph + 1, ph, t, idx);
    }
    inverse_phase<PH, R>(ph, t, bf);
  }
}

// k_cols: one operand per thread; the forward pass covers a (blockIdx.y = 0) and b (= 1)
template <class F, int K, int R, int W, bool INV, int MINB = 1, int EMB = EMB_PLAIN>
__global__ void __launch_bounds__(W * ((1 << K) / R), MINB)
k_cols(F fld0, ColKArgs<F> args) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<K, R>;
  constexpr int NPH = PH::NPH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);

  const int c = threadIdx.x % W;
  const int t = threadIdx.x / W;
  const int64_t inst = blockIdx.x >> cb_log(args);
  const int64_t col = (blockIdx.x & (args.colblocks - 1)) * W + c;
  const int64_t base = inst * args.n + col;
  const int64_t m = args.m;
  const bool second = (!INV) && blockIdx.y == 1;
  const T* src = second ? args.src1 : args.src0;
  T* dst = second ? args.dst1 : args.dst0;
  const ColIdx<PH, W> idx{c};
  const auto fv = field_view(fld0, args, inst);
  const F& fld = select_field(fv, fld0);

  T x[R];
  const int ph_in = INV ? NPH - 1 : 0, ph_out = INV ? 0 : NPH - 1;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int64_t row = PH::ins_t(ph_in, t) + PH::cslot(ph_in, s);
    if constexpr (EMB && !INV) {
      const uint32_t pos = (uint32_t)(col + row * m);
      x[s] = second ? io_load<EMB, true>(src, src_inst<F>(args, inst), pos, (uint32_t)args.n, args.io)
                    : io_load<EMB, false>(src, src_inst<F>(args, inst), pos, (uint32_t)args.n, args.io);
    }
    else x[s] = src[base + row * m];
  }
  if constexpr (!INV) {
    col_forward<PH, K, R, NPH>(x, (T(*)[R]) nullptr, sm, sm, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
      const Tw tw = col_tw<K>(view_twf<F>(fv, args), bit, tb, cs);
      if (second) fld.fwd_bn(x[s0], x[s1], tw);
      else fld.fwd_a(x[s0], x[s1], tw);
    });
  } else {
    col_inverse<PH, K, R, NPH>(x, (T(*)[R]) nullptr, sm, sm, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
      if (bit == K - 1) fld.inv_last(x[s0], x[s1], view_lsi<F>(fv, args), view_lk<F>(fv, args));
      else fld.inv(x[s0], x[s1], col_tw<K>(view_twi<F>(fv, args), bit, tb, cs));
    });
  }
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int64_t row = PH::ins_t(ph_out, t) + PH::cslot(ph_out, s);
    if constexpr (EMB && INV) io_store<EMB>(dst, inst, (uint32_t)(col + row * m), (uint32_t)args.n, x[s], args.io);
    else dst[base + row * m] = x[s];
  }
}

// ------------------------------------------------------------------------------------------
// k_cols_fwd2: the forward column pass for a AND b in the same thread (like k_block): each twiddle
// load serves both splits and every level has twice the independent butterflies per thread, which
// the Goldilocks column pass needs to hide its carry-chain latency (profiles/r01e: k_cols<fwd>
// stalled on "wait" at 2.3 per issue vs 1.2 in k_block).
// ------------------------------------------------------------------------------------------
template <class F, int K, int R, int W, int MINB = 1, int EMB = EMB_PLAIN>
__global__ void __launch_bounds__(W * ((1 << K) / R), MINB)
k_cols_fwd2(F fld0, ColKArgs<F> args) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<K, R>;
  constexpr int NPH = PH::NPH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sma = reinterpret_cast<T*>(smem_raw);
  T* smb = sma + (1 << K) * W;

  const int c = threadIdx.x % W;
  const int t = threadIdx.x / W;
  const int64_t inst = blockIdx.x >> cb_log(args);
  const int64_t col = (blockIdx.x & (args.colblocks - 1)) * W + c;
  const int64_t base = inst * args.n + col;
  const int64_t m = args.m;
  const ColIdx<PH, W> idx{c};
  const auto fv = field_view(fld0, args, inst);
  const F& fld = select_field(fv, fld0);

  constexpr bool OFF32 = sizeof(T) == 8;   // 32-bit row offsets (row m < n <= 2^24) from opaque bases
  const uint32_t mm = (uint32_t)m;
  const T* pa = opaque(args.src0 + base);
  const T* pb = opaque(args.src1 + base);
  T xa[R], xb[R];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int64_t row = PH::ins_t(0, t) + PH::cslot(0, s);
    if constexpr (EMB) {
      const uint32_t pos = (uint32_t)(col + row * m);
      xa[s] = io_load<EMB, false>(args.src0, src_inst<F>(args, inst), pos, (uint32_t)args.n, args.io);
      xb[s] = io_load<EMB, true>(args.src1, src_inst<F>(args, inst), pos, (uint32_t)args.n, args.io);
    } else if constexpr (OFF32) {   // global non-coherent loads (the opaque base alone gives generic LD)
      xa[s] = __ldg(pa + (uint32_t)row * mm);
      xb[s] = __ldg(pb + (uint32_t)row * mm);
    } else {
      xa[s] = args.src0[base + row * m];
      xb[s] = args.src1[base + row * m];
    }
  }
  col_forward<PH, K, R, NPH>(xa, &xb, sma, smb, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
    const Tw tw = col_tw<K>(view_twf<F>(fv, args), bit, tb, cs);
    fld.fwd_a(xa[s0], xa[s1], tw);
    fld.fwd_bn(xb[s0], xb[s1], tw);
  });
  T* qa = opaque(args.dst0 + base);
  T* qb = opaque(args.dst1 + base);
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if constexpr (OFF32) {
      const uint32_t ad = (uint32_t)(PH::ins_t(NPH - 1, t) + PH::cslot(NPH - 1, s)) * mm;
      __stcg(qa + ad, xa[s]);   // st.global (STG), L2 only: read back by the next pass, not this SM
      __stcg(qb + ad, xb[s]);
    } else {
      const int64_t ad = base + (int64_t)(PH::ins_t(NPH - 1, t) + PH::cslot(NPH - 1, s)) * m;
      args.dst0[ad] = xa[s];
      args.dst1[ad] = xb[s];
    }
  }
}

// ------------------------------------------------------------------------------------------
// k_cols_inv2: the inverse column pass with two column groups (c and c + W) per thread, sharing
// every twiddle load and doubling the independent butterflies per level (plain operands).
// ------------------------------------------------------------------------------------------
// VEC: the two column groups of a thread are ADJACENT columns (2c, 2c+1), read and written as one
// 2-element vector access (16 bytes for Goldilocks) instead of two scalar accesses at c and c + W.
template <class T> struct Vec2;
template <> struct Vec2<uint32_t> { using type = uint2; };
template <> struct Vec2<uint64_t> { using type = ulonglong2; };
template <class F, int K, int R, int W, int MINB = 1, int EMB = EMB_PLAIN, bool VEC = false>
__global__ void __launch_bounds__(W * ((1 << K) / R), MINB)
k_cols_inv2(F fld0, ColKArgs<F> args) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<K, R>;
  constexpr int NPH = PH::NPH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sma = reinterpret_cast<T*>(smem_raw);
  T* smb = sma + (1 << K) * W;

  const int c = threadIdx.x % W;
  const int t = threadIdx.x / W;
  const int64_t inst = blockIdx.x >> cb_log(args);     // colblocks = m / (2 W)
  const int64_t base = inst * args.n + (blockIdx.x & (args.colblocks - 1)) * 2 * W + (VEC ? 2 * c : c);
  const int64_t m = args.m;
  const ColIdx<PH, W> idx{c};
  const auto fv = field_view(fld0, args, inst);
  const F& fld = select_field(fv, fld0);
  using V2 = typename Vec2<T>::type;

  T xa[R], xb[R];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int64_t ad = base + (int64_t)(PH::ins_t(NPH - 1, t) + PH::cslot(NPH - 1, s)) * m;
    if constexpr (VEC) {
      const V2 v = *reinterpret_cast<const V2*>(args.src0 + ad);
      xa[s] = v.x;
      xb[s] = v.y;
    } else {
      xa[s] = args.src0[ad];
      xb[s] = args.src0[ad + W];
    }
  }
  col_inverse<PH, K, R, NPH>(xa, &xb, sma, smb, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
    if (bit == K - 1) {
      fld.inv_last(xa[s0], xa[s1], view_lsi<F>(fv, args), view_lk<F>(fv, args));
      fld.inv_last(xb[s0], xb[s1], view_lsi<F>(fv, args), view_lk<F>(fv, args));
    } else {
      const Tw tw = col_tw<K>(view_twi<F>(fv, args), bit, tb, cs);
      fld.inv(xa[s0], xa[s1], tw);
      fld.inv(xb[s0], xb[s1], tw);
    }
  });
  if constexpr (EMB) {   // truncating stores of the polynomial / any-n applications
    const int64_t col = base - inst * args.n;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int64_t pos = col + (int64_t)(PH::ins_t(0, t) + PH::cslot(0, s)) * m;
      io_store<EMB>(args.dst0, inst, (uint32_t)pos, (uint32_t)args.n, xa[s], args.io);
      io_store<EMB>(args.dst0, inst, (uint32_t)(pos + W), (uint32_t)args.n, xb[s], args.io);
    }
  } else {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int64_t ad = base + (int64_t)(PH::ins_t(0, t) + PH::cslot(0, s)) * m;
      if constexpr (VEC) {
        *reinterpret_cast<V2*>(args.dst0 + ad) = V2{xa[s], xb[s]};
      } else {
        args.dst0[ad] = xa[s];
        args.dst0[ad + W] = xb[s];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// k_cols_tma: persistent, TMA-pipelined version of k_cols for plain [batch][n] operands.
//
// Each CTA loops over column tiles (W consecutive columns x all 2^K rows of one instance, one of
// a or b in the forward pass).  One elected thread issues the Tensor Memory Accelerator copy
// (cp.async.bulk.tensor, 3-D map {column, row, instance}) of tile i+1 into the second of two
// shared-memory stages while the CTA transforms tile i, completion signalled through an mbarrier
// with the tile's byte count -- the HBM/L2 latency of the strided column reads is hidden behind
// the integer work instead of stalling each CTA at its start (profiles/r01d: long_scoreboard
// was the top stall of the column passes).  The butterflies, phase exchanges (swizzled smem) and
// stores are those of k_cols.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kTmaBoxRows = 256;   // TMA box extent limit per dimension

template <class F, int K, int R, int W, bool INV, int MINB = 1>
__global__ void __launch_bounds__(W * ((1 << K) / R), MINB)
k_cols_tma(F fld0, ColKArgs<F> args, const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
           int64_t ntiles) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<K, R>;
  constexpr int NPH = PH::NPH;
  constexpr int ROWS = 1 << K;
  constexpr uint32_t TILE_BYTES = (uint32_t)(ROWS * W * sizeof(T));
  // dynamic smem only (a static __shared__ variable would shift the dynamic base off the 128-byte
  // alignment TMA destinations need): [stage 0][stage 1][exchange][2 mbarriers]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // round the base up to 128 bytes in the shared window (the launch adds 128 bytes of slack)
  const uint32_t raw = smem_u32(smem_raw);
  T* stage_buf = reinterpret_cast<T*>(smem_raw + (((raw + 127u) & ~127u) - raw));  // 2 x [ROWS][W] dense
  T* sm = stage_buf + 2 * ROWS * W;                          // exchange buffer, swizzled rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ROWS * W);

  const int c = threadIdx.x % W;
  const int t = threadIdx.x / W;
  const int64_t m = args.m;
  const ColIdx<PH, W> idx{c};

  // tile -> (instance, column block, operand): forward tiles alternate a / b
  auto decode = [&](int64_t tile, int64_t& inst, int64_t& cb, int& second) {
    const int64_t unit = INV ? tile : (tile >> 1);
    second = INV ? 0 : (int)(tile & 1);
    inst = unit >> cb_log(args);
    cb = unit & (args.colblocks - 1);
  };
  auto issue = [&](int64_t tile, int st) {
    int64_t inst, cb;
    int second;
    decode(tile, inst, cb, second);
    const CUtensorMap* map = second ? &map1 : &map0;
    mbar_expect_tx(&bars[st], TILE_BYTES);
#pragma unroll
    for (int rb = 0; rb < ROWS; rb += kTmaBoxRows)
      tma_load_3d(stage_buf + (size_t)st * ROWS * W + (size_t)rb * W, map, (int)(cb * W), rb, (int)inst, &bars[st]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t tile = blockIdx.x;
  if (threadIdx.x == 0 && tile < ntiles) issue(tile, 0);

  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int st = it & 1;
    if (threadIdx.x == 0 && tile + gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of that stage done
      issue(tile + gridDim.x, st ^ 1);
    }
    int64_t inst, cb;
    int second;
    decode(tile, inst, cb, second);
    const int64_t base = inst * args.n + cb * W + c;
    T* dst = second ? args.dst1 : args.dst0;
    const auto fv = field_view(fld0, args, inst);
    const F& fld = select_field(fv, fld0);
    mbar_wait(&bars[st], (uint32_t)((it >> 1) & 1));
    const T* tb_s = stage_buf + (size_t)st * ROWS * W;

    T x[R];
    const int ph_in = INV ? NPH - 1 : 0, ph_out = INV ? 0 : NPH - 1;
#pragma unroll
    for (int s = 0; s < R; ++s) x[s] = tb_s[(PH::ins_t(ph_in, t) + PH::cslot(ph_in, s)) * W + c];
    if constexpr (!INV) {
      col_forward<PH, K, R, NPH>(x, (T(*)[R]) nullptr, sm, sm, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
        const Tw tw = col_tw<K>(view_twf<F>(fv, args), bit, tb, cs);
        if (second) fld.fwd_bn(x[s0], x[s1], tw);
        else fld.fwd_a(x[s0], x[s1], tw);
      });
    } else {
      col_inverse<PH, K, R, NPH>(x, (T(*)[R]) nullptr, sm, sm, t, idx, [&](int s0, int s1, int bit, int tb, int cs) {
        if (bit == K - 1) fld.inv_last(x[s0], x[s1], view_lsi<F>(fv, args), view_lk<F>(fv, args));
        else fld.inv(x[s0], x[s1], col_tw<K>(view_twi<F>(fv, args), bit, tb, cs));
      });
    }
#pragma unroll
    for (int s = 0; s < R; ++s) dst[base + (int64_t)(PH::ins_t(ph_out, t) + PH::cslot(ph_out, s)) * m] = x[s];
    __syncthreads();   // stage st and the exchange buffer are free for the next issue / tile
  }
}


// ------------------------------------------------------------------------------------------
// k_block_pipe: the 32-bit sub-problem kernel with its operand loads taken off the critical path.
//
// One CTA per SM of 2 x (2^M / R) threads: two independent halves share the staged twiddle slice
// of sub-block E and each walks its own sequence of instances of E.  A half's
// a' and b' slices (2^M contiguous elements each) are brought into a shared-memory stage by the
// Tensor Memory Accelerator's bulk copy (cp.async.bulk, mbarrier with the byte count) one
// instance AHEAD: while the half transforms instance j from registers, the copy of instance j + 1
// is in flight, so the global-load latency that stalled k_block at every instance start
// (long_scoreboard, profiles/r01n_ncu_full_S1.txt) overlaps the arithmetic.  The halves synchronise
// their exchanges with their own named barriers (bar.sync 1 / 2), so one never waits for the other.
// Shared memory: twiddles 2 x 2^M Tw + per half (stage 2 x 2^M T, exchange 2 x 2^M T) + mbarriers.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <class F, int M, int R>
__global__ void __launch_bounds__(2 * (1 << M) / R, 1)
k_block_pipe(F fld0, BlockKArgs<F> args) {
  pdl_entry();
  using T = typename F::T;
  using Tw = typename F::Tw;
  using PH = Phases<M, R>;
  constexpr int m = 1 << M;
  constexpr int TT = PH::T;
  constexpr int NPH = PH::NPH;
  constexpr uint32_t SLICE = (uint32_t)(m * sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tw* twsf = reinterpret_cast<Tw*>(smem_raw);
  Tw* twsi = twsf + m;
  const int half = threadIdx.x / TT;
  const int t = threadIdx.x % TT;
  T* stage_a = reinterpret_cast<T*>(twsi + m) + (size_t)half * 4 * m;   // [stage a | stage b | xa | xb]
  T* stage_b = stage_a + m;
  T* sa = stage_a + 2 * m;
  T* sb = stage_a + 3 * m;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<T*>(twsi + m) + (size_t)8 * m);
  const NamedSync hsync{1 + half, TT};
  auto idx = [](int base_part, int slot_part) { return swz<R, T>(base_part) ^ swz<R, T>(slot_part); };

  const int k = args.k;
  const int64_t batch = args.units >> k;
  const int nseq = args.seq;                         // instances per half
  const int E = (int)(blockIdx.x & ((1u << k) - 1));
  const int64_t first = (int64_t)(blockIdx.x >> k) * 2 * nseq;   // the CTA's first instance
  const auto fv = field_view(fld0, args, first);     // one prime per CTA (launcher)
  const F& fld = select_field(fv, fld0);
  auto inst_of = [&](int j) { return first + 2 * (int64_t)j + half; };
  auto src_a = [&](int64_t inst) { return args.a + ((inst << k) + E) * (int64_t)m; };
  auto src_b = [&](int64_t inst) { return args.b + ((inst << k) + E) * (int64_t)m; };
  auto issue = [&](int64_t inst) {
    mbar_expect_tx(&bars[half], 2 * SLICE);
    bulk_load(stage_a, src_a(inst), SLICE, &bars[half]);
    bulk_load(stage_b, src_b(inst), SLICE, &bars[half]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // twiddle slice of sub-block E (all threads), as k_block's staging
  for (int h = threadIdx.x + 1; h < m; h += blockDim.x) {
    const int j = 31 - __clz(h);
    const int g = (1 << (k + j)) + (E << j) + (h - (1 << j));
    twsf[tw_swz(h)] = view_twf<F>(fv, args)[g];
    twsi[tw_swz(h)] = view_twi<F>(fv, args)[g];
  }
  __syncthreads();
  if (t == 0 && inst_of(0) < batch) issue(inst_of(0));

  auto tw_st = [&](const Tw* staged, int bit, int tb, int cs) -> Tw {
    return staged[tw_swz(1 << (M - 1 - bit)) ^ tw_swz(tb >> (bit + 1)) ^ tw_swz(cs >> (bit + 1))];
  };
  for (int j = 0; j < nseq; ++j) {
    const int64_t inst = inst_of(j);
    if (inst >= batch) break;                         // uniform per half
    mbar_wait(&bars[half], (uint32_t)(j & 1));
    T xa[R], xb[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int ad = PH::ins_t(0, t) + PH::cslot(0, s);
      xa[s] = stage_a[ad];
      xb[s] = stage_b[ad];
    }
    hsync();                                          // the half has read the stage: refill it
    if (t == 0 && inst_of(j + 1) < batch && j + 1 < nseq) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(inst_of(j + 1));
    }
#pragma unroll
    for (int ph = 0; ph < NPH; ++ph) {
      if (ph > 0) exchange2<PH, R>(xa, xb, sa, sb, ph - 1, ph, t, idx, hsync);
      forward_phase<PH, R>(ph, t, [&](int s0, int s1, int bit, int tb, int cs) {
        const Tw tw = tw_st(twsf, bit, tb, cs);
        fld.fwd_a(xa[s0], xa[s1], tw);
        fld.fwd_b(xb[s0], xb[s1], tw);
      });
    }
    T xm[R];
    leaves<PH, F, R>(fld, xm, xa, xb, E, t);
#pragma unroll
    for (int ph = NPH - 1; ph >= 0; --ph) {
      if (ph < NPH - 1) exchange<PH, R>(xm, sa, ph + 1, ph, t, idx, hsync);
      inverse_phase<PH, R>(ph, t, [&](int s0, int s1, int bit, int tb, int cs) {
        fld.inv(xm[s0], xm[s1], tw_st(twsi, bit, tb, cs));
      });
    }
    T* out = args.out + ((inst << k) + E) * (int64_t)m;
#pragma unroll
    for (int s = 0; s < R; ++s) out[PH::ins_t(0, t) + PH::cslot(0, s)] = xm[s];
  }
}

}  // namespace fcirc

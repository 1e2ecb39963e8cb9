// matvec_impl.cuh — launch tables and the pass schedule of the f-circulant product (SURVEY §8(a)
// row H6), instantiated once per field by matvec_u32.cu / matvec_gold.cu.
//
//   n <= 2^MMAX  : one k_block launch with k = 0 (fused: one HBM read of a and b, one write of c)
//   n >  2^MMAX  : per chunk of instances sized to stay L2-resident
//                    k_cols<fwd>  top K = L - MMAX levels of a and b  -> a' (in c), b' (workspace)
//                    k_block      the 2^K sub-products of size 2^MMAX  -> M (in c, in place)
//                    k_cols<inv>  top K inverse levels, 1/n scaling     -> c (in place)
#pragma once
#include <algorithm>
#include <cstdint>
#include <utility>

#include <cudaTypedefs.h>

#include "../../include/fcirc.h"
#include "fcirc_kernels.cuh"
#include "runtime.h"

namespace fcirc {

template <class F> struct FTraits;
template <> struct FTraits<FieldU32> {
  static constexpr int MMAX = 13;   // 2 x 2^13 x 4 B data + 2 x 2^13 x 8 B staged twiddles = 192 KB smem
  static constexpr int MPREF = 12;  // 96 KB: two CTAs per SM
  static constexpr const char* RB = "U32_RB";
  static constexpr const char* RBF = "U32_RBF";
  static constexpr const char* SEQ = "U32_SEQ";
  static constexpr const char* RC = "U32_RC";
  static constexpr const char* MS = "U32_MSPLIT";
  static constexpr int TMA_MIN_K = 9;   // TMA inverse column passes from this depth on; below it
                                        // k_cols_inv2 measured faster (profiles/r01e_sweep_inv2.txt)
};
template <> struct FTraits<FieldU32M> : FTraits<FieldU32> {};   // multi-prime launches (bigint)
template <> struct FTraits<FieldGold> {
  static constexpr int MMAX = 13;   // 2 x 2^13 x 8 B = 128 KB smem per sub-problem
  static constexpr int MPREF = 12;  // 64 KB: two CTAs per SM
  static constexpr const char* RB = "GOLD_RB";
  static constexpr const char* RBF = "GOLD_RBF";
  static constexpr const char* SEQ = "GOLD_SEQ";
  static constexpr const char* RC = "GOLD_RC";
  static constexpr const char* MS = "GOLD_MSPLIT";
  static constexpr int TMA_MIN_K = 9;
};
template <> struct FTraits<FieldM31x2> {      // the paper's ring, 8-byte packed elements (as Goldilocks)
  static constexpr int MMAX = 13;
  static constexpr int MPREF = 12;
  static constexpr const char* RB = "M31_RB";
  static constexpr const char* RBF = "M31_RBF";
  static constexpr const char* SEQ = "M31_SEQ";
  static constexpr const char* RC = "M31_RC";
  static constexpr const char* MS = "M31_MSPLIT";
  static constexpr int TMA_MIN_K = 9;
};
constexpr int KMAX = 11;

// elements per thread (registers) for a transform of 2^M points; threads = 2^M / R
template <int RR> constexpr int rsel(int M) { return M < 4 ? (1 << M) : RR; }
template <int RR> constexpr int ipcsel(int M) {
  return ((1 << M) / rsel<RR>(M)) >= 128 ? 1 : 128 / ((1 << M) / rsel<RR>(M));
}
// consecutive columns per k_cols CTA: >= 8 for 64-byte row segments, ~256 threads per CTA
template <int RR> constexpr int wsel(int K) {
  return (256 * rsel<RR>(K)) >> K < 8 ? 8 : ((256 * rsel<RR>(K)) >> K);
}

// k_block_pipe (32-bit fields, staged sub-problem launches of 2^12 points at R = 8): two instance
// streams per CTA with bulk-copy prefetch of the next instance's operands (fcirc_kernels.cuh).
// FCIRC_U32_PIPE=0 disables it; FCIRC_U32_PSEQ = instances per half (default 8).
template <class F, int M, int R>
static int launch_block_pipe(const F& fld, const BlockKArgs<F>& args, cudaStream_t st) {
  using E = typename F::T;
  using Tw = typename F::Tw;
  constexpr int T = (1 << M) / R;
  const size_t smem = (size_t)2 * (1 << M) * sizeof(Tw) + (size_t)8 * (1 << M) * sizeof(E) + 16;
  auto kern = k_block_pipe<F, M, R>;
  static std::atomic<uint32_t> attr_mask{0};
  if (!smem_optin((const void*)kern, smem, attr_mask)) return FCIRC_ECUDA;
  const int64_t batch = args.units >> args.k;
  static const int knob_seq = std::max(1, knob("U32_PSEQ", 8));
  int seq = 1;
  while (seq * 2 <= knob_seq && 2 * seq * 2 <= batch) seq *= 2;
  if constexpr (kMulti<F>)   // the CTA's 2 seq instances inside one prime
    while (seq > 1 && (args.mp.per % (2 * seq) != 0 || args.mp.inst0 % (2 * seq) != 0)) seq >>= 1;
  BlockKArgs<F> a2 = args;
  a2.seq = seq;
  const int64_t grid = ((batch + 2 * seq - 1) / (2 * seq)) << args.k;
  prof_begin(1, st);
  launch_k(kern, (unsigned)grid, 2 * T, smem, st, fld, a2);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// An application call's embedding mode as a compile-time constant: the first / last pass kernels are
// instantiated per mode (TRUNC: only the truncating modes, whose inverse pass stores through the
// embedding; limbs only for the 32-bit fields).
template <class F, bool TRUNC = false, class Fn>
static int with_emb(int mode, Fn&& fn) {
  switch (mode) {
    case EMB_POLY: return fn(std::integral_constant<int, EMB_POLY>{});
    case EMB_ANYN: return fn(std::integral_constant<int, EMB_ANYN>{});
    case EMB_LIMBS:
      if constexpr (!TRUNC && sizeof(typename F::T) == 4) return fn(std::integral_constant<int, EMB_LIMBS>{});
      return FCIRC_EINVAL;
    default: return FCIRC_EINVAL;
  }
}

template <class F, int M, int RR, int EMB, bool TWS>
static int launch_block_t(const F& fld, const BlockKArgs<F>& args, cudaStream_t st) {
  constexpr int R = rsel<RR>(M), IPC = ipcsel<RR>(M);
  constexpr int T = (1 << M) / R;
  using E = typename F::T;
  constexpr int PM = 1 << M;  // swizzled, unpadded (fcirc_kernels.cuh swz)
  if constexpr (TWS && !EMB && sizeof(E) == 4 && M == 12 && R == 8) {
    // measured against this kernel: S1 +1.3 %, C3 -4..8 %, C5 +-0 (profiles/r02d_ab_pipe.txt): off
    // by default
    static const int use_pipe = knob("U32_PIPE", 0);
    const bool aligned = ((uintptr_t)args.a & 15) == 0 && ((uintptr_t)args.b & 15) == 0;
    bool pairs_in_one_prime = true;   // a CTA's two halves start in one prime
    if constexpr (kMulti<F>) pairs_in_one_prime = args.mp.per % 2 == 0 && args.mp.inst0 % 2 == 0;
    if (use_pipe && args.k > 0 && aligned && pairs_in_one_prime) return launch_block_pipe<F, M, R>(fld, args, st);
  }
  const size_t smem = (size_t)IPC * 2 * PM * sizeof(E) + (TWS ? (size_t)2 * (1 << M) * sizeof(typename F::Tw) : 0);
  // occupancy target: 1024 resident threads per SM (register cap 64) for R <= 8, and for R = 16
  // with 32-bit elements when the twiddles are not staged (plain loads, M = 12: fits 64 registers
  // with at most a 16-byte spill; measured C2 +5.6 %, profiles/r01h_sweep_u32_r16.txt); 512 otherwise (cap 128: without a floor ptxas spends ~190
  // registers and halves the resident warps; with staged twiddles shared memory admits only two
  // 256-thread CTAs per SM anyway, and a 64-register cap would only add spills)
  constexpr int TGT = (RR <= 8 || (sizeof(E) == 4 && !TWS && !EMB && M == 12)) ? 1024 : 512;
  constexpr int MINB = (T * IPC < TGT) ? TGT / (T * IPC) : 1;
  auto kern = k_block<F, M, R, IPC, MINB, EMB, TWS>;
  int variant = 0;
  if constexpr (M == 12 && R == 8 && !EMB) {
    // FCIRC_SHFL=1: the last exchange of sub-problem launches as an in-warp lane transpose (A/B only;
    // measured slower)
    static const int shf = knob("SHFL", 0);
    if (shf && args.k > 0) { kern = k_block<F, M, R, IPC, MINB, EMB, TWS, true>; variant = 1; }
  }
  static std::atomic<uint32_t> attr_mask[2];   // opt-in shared memory once per (kernel, device)
  if (!smem_optin((const void*)kern, smem, attr_mask[variant]))
    return FCIRC_ECUDA;
  const int64_t batch = args.units >> args.k;
  BlockKArgs<F> a2 = args;
  // staged sub-problem launches: each CTA walks seq instance groups of one sub-block, staging its
  // twiddle slice once (FCIRC_<field>_SEQ; default: the largest power of two <= 16 that still
  // leaves >= 1024 CTAs, about 3.5 waves of resident CTAs -- measured best for S1 (16), C3 (8)
  // and C5 (1), profiles/r01i_sweep_seq.txt)
  if constexpr (TWS) {   // (unstaged Goldilocks launches measured slower with seq > 1)
    static const int knob_seq = knob(FTraits<F>::SEQ, 0);
    const int64_t groups = (batch + IPC - 1) / IPC;
    int seq = 1;
    if (args.k > 0) {
      if (knob_seq > 0) seq = knob_seq;
      else
        while (seq < 16 && ((groups / (2 * seq)) << args.k) >= 1024) seq *= 2;
    }
    a2.seq = (int)std::min<int64_t>(seq, groups);
    // several primes in one launch: a staged CTA's instances must stay inside one prime
    if constexpr (kMulti<F>)
      while (a2.seq > 1 && ((args.mp.per % ((int64_t)IPC * a2.seq)) != 0 || (args.mp.inst0 % ((int64_t)IPC * a2.seq)) != 0))
        a2.seq >>= 1;
  }
  const int64_t per_cta = (int64_t)IPC * a2.seq;
  const int64_t grid = ((batch + per_cta - 1) / per_cta) << args.k;
  prof_begin(args.k == 0 ? 0 : 1, st);
  launch_k(kern, (unsigned)grid, T * IPC, smem, st, fld, a2);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// The 32-bit fields stage their twiddle slices in smem for sub-problem launches (k > 0), and for
// fused launches of a small batch (latency-bound: one coalesced table load per CTA instead of a
// dependent L2 round trip per phase); large fused batches share the table through L1/L2 instead.
template <class F, int M, int RR, int EMB = EMB_PLAIN>
static int launch_block(const F& fld, const BlockKArgs<F>& args, cudaStream_t st) {
  if constexpr (TwStage<F, M>::value && !EMB) {
    bool one_prime_per_cta = true;   // multi-prime: a staged CTA's IPC instances inside one prime
    if constexpr (kMulti<F>)
      one_prime_per_cta = args.mp.per % ipcsel<RR>(M) == 0 && args.mp.inst0 % ipcsel<RR>(M) == 0;
    // sub-problem launches read their twiddles through L1 / L2 (R = 16 at 1024 threads/SM): measured
    // faster than staging them (512 threads/SM) once R = 16 won (profiles/r02l_ab_tma_stage.txt);
    // FCIRC_U32_STAGE=1 restores the staged kernel
    static const int stage = knob("U32_STAGE", 0);
    if ((args.k > 0 || args.units <= 64) && one_prime_per_cta && (stage || args.k == 0))
      return launch_block_t<F, M, RR, EMB_PLAIN, true>(fld, args, st);
  }
  return launch_block_t<F, M, RR, EMB, false>(fld, args, st);
}

template <class F, int K, bool INV, int RR, int EMB = EMB_PLAIN>
static int launch_cols(const F& fld, ColKArgs<F> args, int64_t instances, cudaStream_t st) {
  constexpr int R = rsel<RR>(K), W = wsel<RR>(K);
  constexpr int threads = W * ((1 << K) / R);
  using E = typename F::T;
  const size_t smem = (size_t)(1 << K) * W * sizeof(E);
  constexpr int MINB = (threads < (RR <= 8 ? 1024 : 512)) ? (RR <= 8 ? 1024 : 512) / threads : 1;
  auto kern = k_cols<F, K, R, W, INV, MINB, EMB>;
  static std::atomic<uint32_t> attr_mask{0};   // opt-in shared memory once per (kernel, device)
  if (!smem_optin((const void*)kern, smem, attr_mask)) return FCIRC_ECUDA;
  args.colblocks = args.m / W;
  args.units = instances * args.colblocks;
  dim3 grid((unsigned)args.units, INV ? 1 : 2);
  prof_begin(INV ? 3 : 2, st);
  launch_k(kern, grid, threads, smem, st, fld, args);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// dual forward column pass (a and b per thread)
template <class F, int K, int RR, int EMB = EMB_PLAIN>
static int launch_cols_fwd2(const F& fld, ColKArgs<F> args, int64_t instances, cudaStream_t st) {
  constexpr int R = rsel<RR>(K), W = wsel<RR>(K);
  constexpr int threads = W * ((1 << K) / R);
  using E = typename F::T;
  const size_t smem = (size_t)2 * (1 << K) * W * sizeof(E);
  // 32-bit elements fit R = 16 in 64 registers here: 1024 threads/SM (C3 forward column pass -9 %,
  // S1 -2 %; the inverse kernel would spill, profiles/r01j_sweep_cols1024.txt)
  constexpr int TGT = (RR <= 8 || sizeof(E) == 4) ? 1024 : 512;
  constexpr int MINB = (threads < TGT) ? TGT / threads : 1;
  auto kern = k_cols_fwd2<F, K, R, W, MINB, EMB>;
  static std::atomic<uint32_t> attr_mask{0};   // opt-in shared memory once per (kernel, device)
  if (!smem_optin((const void*)kern, smem, attr_mask)) return FCIRC_ECUDA;
  args.colblocks = args.m / W;
  args.units = instances * args.colblocks;
  prof_begin(2, st);
  launch_k(kern, (unsigned)args.units, threads, smem, st, fld, args);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// inverse column pass, two column groups per thread (plain operands; needs m >= 2 W)
template <class F, int K, int RR, int EMB = EMB_PLAIN>
static int launch_cols_inv2(const F& fld, ColKArgs<F> args, int64_t instances, cudaStream_t st) {
  constexpr int R = rsel<RR>(K), W = wsel<RR>(K);
  constexpr int threads = W * ((1 << K) / R);
  using E = typename F::T;
  const size_t smem = (size_t)2 * (1 << K) * W * sizeof(E);
  // 32-bit R = 16: 768 resident threads (<= 85 registers) instead of 512 (96 registers, 23 % of the
  // warp slots active, latency-bound: profiles/r02f_ncu_full_S1.txt)
  constexpr int TGT = RR <= 8 ? 1024 : (sizeof(E) == 4 ? 768 : 512);
  constexpr int MINB = (threads < TGT) ? TGT / threads : 1;
  auto kern = k_cols_inv2<F, K, R, W, MINB, EMB>;
  if constexpr (!EMB) {
    // adjacent column pairs as one 2-element vector access (16 bytes for the 8-byte fields; the
    // north-star's 128-bit accesses): measured equal to the scalar pair at C4 n = 2^20
    // (profiles/r02e_gold_ab_shfl_vec.txt), default on when the base is 16-byte aligned
    static const int vec = knob("VEC", 1);
    if (vec && ((uintptr_t)args.src0 & 15) == 0 && ((uintptr_t)args.dst0 & 15) == 0)
      kern = k_cols_inv2<F, K, R, W, MINB, EMB, true>;
  }
  static std::atomic<uint32_t> attr_mask[2];   // opt-in shared memory once per (kernel, device)
  if (!smem_optin((const void*)kern, smem, attr_mask[kern == k_cols_inv2<F, K, R, W, MINB, EMB> ? 0 : 1]))
    return FCIRC_ECUDA;
  args.colblocks = args.m / (2 * W);
  args.units = instances * args.colblocks;
  prof_begin(3, st);
  launch_k(kern, (unsigned)args.units, threads, smem, st, fld, args);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// ---- TMA-pipelined column passes (k_cols_tma): tensor maps through the driver entry point
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}

// 3-D view {column < m, row < 2^K, instance} of a [instances][n] array, box {W, min(2^K, 256), 1}
template <class E>
static bool make_col_map(CUtensorMap* map, const void* base, int64_t m, int K, int64_t instances, int W) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)m, (cuuint64_t)1 << K, (cuuint64_t)instances};
  const cuuint64_t strides[2] = {(cuuint64_t)m * sizeof(E), ((cuuint64_t)m << K) * sizeof(E)};
  const cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)std::min(1 << K, kTmaBoxRows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, sizeof(E) == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 3,
             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class F, int K, bool INV, int RR>
static int launch_cols_tma(const F& fld, ColKArgs<F> args, int64_t instances, cudaStream_t st) {
  constexpr int R = rsel<RR>(K), W = wsel<RR>(K);
  constexpr int threads = W * ((1 << K) / R);
  using E = typename F::T;
  // two TMA stages + exchange buffer + 2 mbarriers + 128 bytes of alignment slack
  const size_t smem = (size_t)3 * (1 << K) * W * sizeof(E) + 16 + 128;
  constexpr int MINB = (threads < (RR <= 8 ? 1024 : 512)) ? (RR <= 8 ? 1024 : 512) / threads : 1;
  auto kern = k_cols_tma<F, K, R, W, INV, MINB>;
  static std::atomic<uint32_t> attr_mask{0};   // opt-in shared memory once per (kernel, device)
  if (!smem_optin((const void*)kern, smem, attr_mask)) return FCIRC_ECUDA;
  int occ = 0;   // resident CTAs per SM (after the opt-in on this device)
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1)
    return FCIRC_ECUDA;
  args.colblocks = args.m / W;
  args.units = instances * args.colblocks;
  CUtensorMap m0, m1;
  if (!make_col_map<E>(&m0, args.src0, args.m, K, instances, W)) return FCIRC_ECUDA;
  if (!INV && !make_col_map<E>(&m1, args.src1, args.m, K, instances, W)) return FCIRC_ECUDA;
  if (INV) m1 = m0;
  const int64_t ntiles = args.units * (INV ? 1 : 2);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * occ);
  prof_begin(INV ? 3 : 2, st);
  launch_k(kern, (unsigned)grid, threads, smem, st, fld, args, m0, m1, ntiles);
  prof_end(st);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

// Register-blocking variants: the two largest sub-problem sizes and the deep column
// transforms are instantiated with R = 16, 8 and 4 elements per thread, selected by the runtime
// knobs FCIRC_<field>_RB / _RC (defaults from the measured sweep, profiles/r01c_sweep.txt).
// Smaller R = more threads per sub-problem and fewer registers per thread: more resident warps to
// hide the latency of the carry chains, at the price of more shared-memory exchange phases.
template <class F> struct RDefault;
// RB: sub-problem launches (and the staged-twiddle small fused ones); RBF: fused launches of a large
// batch with plain twiddle loads (u32: R = 16 at 1024 threads/SM, C2 +5 %; the staged sub-problem
// kernels measured 0.1-0.5 % faster with R = 8, profiles/r01h_sweep_u32_r16.txt)
template <> struct RDefault<FieldU32> { static constexpr int RB = 16, RBF = 16, RC = 16; };   // RB 16: r02i re-sweep
template <> struct RDefault<FieldU32M> : RDefault<FieldU32> {};
template <> struct RDefault<FieldGold> { static constexpr int RB = 8, RBF = 8, RC = 8; };
template <> struct RDefault<FieldM31x2> { static constexpr int RB = 8, RBF = 8, RC = 8; };

template <class F, int M>
static int launch_block_r(const F& fld, const BlockKArgs<F>& args, cudaStream_t st) {
  // the application embeddings (fused path only) use one variant: the default R
  if (args.k == 0 && args.io.mode != EMB_PLAIN)
    return with_emb<F>(args.io.mode, [&](auto md) { return launch_block<F, M, RDefault<F>::RB, decltype(md)::value>(fld, args, st); });
  // latency-bound small fused batches (C1: one 1024-point product): 4 elements per thread, i.e.
  // more and shorter dependency chains (C1 7.5 -> 5.6 us per step, profiles/r01m_sweep_c1_small_r.txt)
  if constexpr (M >= 8 && M <= 10) {
    static const int rs = knob("SMALL_R", 4);
    if (args.k == 0 && args.units <= 64) {
      if (rs == 4) return launch_block<F, M, 4>(fld, args, st);
      if (rs == 8) return launch_block<F, M, 8>(fld, args, st);
    }
  }
  if constexpr (M >= FTraits<F>::MMAX - 2) {
    static const int rb = knob(FTraits<F>::RB, RDefault<F>::RB);
    static const int rbf = knob(FTraits<F>::RBF, RDefault<F>::RBF);
    const bool fused_plain = args.k == 0 && !(TwStage<F, M>::value && args.units <= 64);
    const int r = fused_plain ? rbf : rb;
    if (r == 8) return launch_block<F, M, 8>(fld, args, st);
    if constexpr ((1 << M) / 4 <= 1024)  // one sub-problem per CTA: at most 1024 threads
      if (r == 4) return launch_block<F, M, 4>(fld, args, st);
  }
  return launch_block<F, M, 16>(fld, args, st);
}

// Column-pass selection (measured, profiles/r01e_sweep_cols2.txt):
//   forward, plain, K >= 6      -> k_cols_fwd2 (a and b per thread)        FCIRC_COLS2=0 disables
//   forward, embedded operands  -> k_cols_fwd2<EMB> (polynomial, any-n, and limbs: C5's forward
//                                  column pass 0.118 -> 0.090 ms at 1024 threads/SM, r01l sweep)
//   inverse, K >= TMA_MIN_K     -> k_cols_tma (persistent, TMA double-buffered)  FCIRC_TMA=0 disables
//   inverse, 6 <= K < TMA_MIN_K -> k_cols_inv2 (two column groups per thread)   FCIRC_INV2=0 disables
//   otherwise                   -> k_cols (R = 16, or the FCIRC_<field>_RC variant)
template <class F, int K, bool INV>
static int launch_cols_r(const F& fld, const ColKArgs<F>& args, int64_t inst, cudaStream_t st) {
  static const int use_tma = knob("TMA", 1);
  static const int use_fwd2 = knob("COLS2", 1);
  static const int r = knob(FTraits<F>::RC, RDefault<F>::RC);
  using E = typename F::T;
  const int mode = args.io.mode;
  if constexpr (!INV && K >= 4 && K <= 10) {
    if (use_fwd2 && mode != EMB_PLAIN)
      return with_emb<F>(mode, [&](auto md) { return launch_cols_fwd2<F, K, 16, decltype(md)::value>(fld, args, inst, st); });
    if (use_fwd2 && mode == EMB_PLAIN && K >= 6) {
      if (r == 8) return launch_cols_fwd2<F, K, 8>(fld, args, inst, st);
      return launch_cols_fwd2<F, K, 16>(fld, args, inst, st);
    }
  }
  // application embeddings: the forward pass reads embedded operands (above); the inverse pass of
  // a truncating embedding (polynomial, any-n) stores through EMB; a limb embedding's inverse
  // output is a plain [batch][n] array and takes the plain selection below
  if (!INV && mode != EMB_PLAIN)
    return with_emb<F>(mode, [&](auto md) { return launch_cols<F, K, INV, 16, decltype(md)::value>(fld, args, inst, st); });
  if (INV && emb_truncates(mode)) {
    if constexpr (K >= 6 && K <= 10)
      if (args.m >= 2 * wsel<16>(K))
        return with_emb<F, true>(mode, [&](auto md) { return launch_cols_inv2<F, K, 16, decltype(md)::value>(fld, args, inst, st); });
    return with_emb<F, true>(mode, [&](auto md) { return launch_cols<F, K, INV, 16, decltype(md)::value>(fld, args, inst, st); });
  }
  static const int use_inv2 = knob("INV2", 1);
  // depth from which the inverse column pass takes the TMA pipeline (FCIRC_TMA_MIN_K; instantiated
  // from K = 7 on so the boundary can be re-swept without a rebuild)
  static const int tma_min_k = knob("TMA_MIN_K", FTraits<F>::TMA_MIN_K);
  if constexpr (INV && K >= 6 && K <= 10) {
    // two column groups per thread below the TMA depth (and whenever FCIRC_TMA=0)
    if (use_inv2 && (!use_tma || K < tma_min_k) && args.m >= 2 * wsel<16>(K)) {
      if (r == 8) return launch_cols_inv2<F, K, 8>(fld, args, inst, st);
      return launch_cols_inv2<F, K, 16>(fld, args, inst, st);
    }
  }
  // TMA pipeline when two stages + the exchange buffer fit in shared memory and the tensor-map bases
  // are 16-byte aligned (cuTensorMapEncodeTiled's requirement; an offset view of a caller's tensor
  // may be only element-aligned and then takes the plain column kernels below)
  if constexpr (K >= 7 && 3 * (1 << K) * wsel<16>(K) * sizeof(E) <= 200 * 1024) {
    const bool aligned = ((uintptr_t)args.src0 & 15) == 0 && (INV || ((uintptr_t)args.src1 & 15) == 0);
    if (use_tma && aligned && K >= tma_min_k) {
      if constexpr (K <= 10)
        if (r == 8) return launch_cols_tma<F, K, INV, 8>(fld, args, inst, st);
      return launch_cols_tma<F, K, INV, 16>(fld, args, inst, st);
    }
  }
  if constexpr (K >= 6 && K <= 10) {  // K = 11 with R = 8 would need 2048 threads
    if (r == 8) return launch_cols<F, K, INV, 8>(fld, args, inst, st);
    if constexpr (K <= 9)
      if (r == 4) return launch_cols<F, K, INV, 4>(fld, args, inst, st);
  }
  return launch_cols<F, K, INV, 16>(fld, args, inst, st);
}

template <class F, int... Ms>
static int dispatch_block(int M, const F& fld, const BlockKArgs<F>& args, cudaStream_t st,
                          std::integer_sequence<int, Ms...>) {
  int rc = FCIRC_EINVAL;
  ((M == Ms ? (rc = launch_block_r<F, Ms>(fld, args, st), 0) : 0), ...);
  return rc;
}

template <class F, bool INV, int... Ks>
static int dispatch_cols(int K, const F& fld, const ColKArgs<F>& args, int64_t inst, cudaStream_t st,
                         std::integer_sequence<int, Ks...>) {
  int rc = FCIRC_EINVAL;
  ((K == Ks + 1 ? (rc = launch_cols_r<F, Ks + 1, INV>(fld, args, inst, st), 0) : 0), ...);
  return rc;
}

// On-chip sub-problem size for a product of order 2^L: the preferred split (FCIRC_<field>_MSPLIT in
// [MMAX-2, MMAX], default FTraits::MPREF; u32 prefers 2^12 = two CTAs per SM over 2^13 = one,
// profiles/r01d), grown
// up to MMAX only when the column passes would need more than KMAX levels.
template <class F>
static int msplit(int L) {
  static const int pref = std::min(FTraits<F>::MMAX,
                                   std::max(FTraits<F>::MMAX - 2, knob(FTraits<F>::MS, FTraits<F>::MPREF)));
  return std::min(FTraits<F>::MMAX, std::max(pref, L - KMAX));
}

// mp (FieldU32M only): several primes in one launch per pass -- instance j of the
// [batch][n] output belongs to prime j / mp->per and reads the operands of instance j % mp->per
template <class F>
static int run_matvec(const F& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                      int64_t batch, cudaStream_t st, int dev, const EmbedIO& io, const MultiPrime* mp = nullptr) {
  using E = typename F::T;
  using Tw = typename F::Tw;
  const int MMAX = msplit<F>(L);
  const Tw* twf = (const Tw*)dp.twf;
  const Tw* twi = (const Tw*)dp.twi;
  Tw lsi, lk;
  if constexpr (sizeof(E) == 4) { lsi = dp.last_si32; lk = dp.last_k32; }
  else { lsi = dp.last_si64; lk = dp.last_k64; }
  const int64_t n = (int64_t)1 << L;
  const MultiPrime mp1 = mp ? *mp : MultiPrime{};
  if (L <= MMAX) {
    BlockKArgs<F> ba;
    static_cast<BlockArgs<F>&>(ba) = BlockArgs<F>{(const E*)a, (const E*)b, (E*)c, batch, 0, twf, twi, lsi, lk, io};
    if constexpr (kMulti<F>) ba.mp = mp1;
    return dispatch_block<F>(L, fld, ba, st, std::make_integer_sequence<int, FTraits<F>::MMAX + 1>{});
  }
  const int K = L - MMAX;
  if (K > KMAX) return FCIRC_ESIZE;
  const bool plain = io.mode == EMB_PLAIN;
  const int64_t per_inst = 2 * n * (int64_t)sizeof(E);
  int64_t C = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)chunk_bytes() / per_inst));
  // plain: a' lives in c, b' in the workspace; embedded inputs: a' and b' both in the workspace
  void* ws;
  int rc = ws_alloc(dev, st, (size_t)((plain ? 1 : 2) * C * n) * sizeof(E), &ws);
  if (rc) return rc;
  struct Free { void* p; cudaStream_t s; ~Free() { ws_free(p, s); } } free_ws{ws, st};
  // instance strides of the caller's arrays (elements of E; 32-bit words for EMB_LIMBS)
  const int64_t sa = plain ? n : io.na, sb = plain ? n : io.nb, sc = emb_truncates(io.mode) ? io.nc : n;
  for (int64_t i0 = 0; i0 < batch; i0 += C) {
    const int64_t cc = std::min<int64_t>(C, batch - i0);
    // multi-prime launches index the caller's operands by the global instance (src_inst), so their
    // source pointers are not advanced per chunk; the chunk's first global instance is mp.inst0
    MultiPrime mpc = mp1;
    mpc.inst0 = i0;
    const E* ai = (const E*)a + (mp1.n > 1 ? 0 : i0 * sa);
    const E* bi = (const E*)b + (mp1.n > 1 ? 0 : i0 * sb);
    E* ci = (E*)c + i0 * sc;
    E* ap = plain ? ci : (E*)ws;
    E* bw = plain ? (E*)ws : (E*)ws + C * n;
    ColKArgs<F> fa;
    static_cast<ColArgs<F>&>(fa) = ColArgs<F>{ai, bi, ap, bw, n >> K, n, 0, 0, twf, twi, lsi, lk, io};
    if constexpr (kMulti<F>) fa.mp = mpc;
    rc = dispatch_cols<F, false>(K, fld, fa, cc, st, std::make_integer_sequence<int, KMAX>{});
    if (rc) return rc;
    BlockKArgs<F> ba;
    static_cast<BlockArgs<F>&>(ba) = BlockArgs<F>{ap, bw, ap, cc << K, K, twf, twi, lsi, lk, EmbedIO{}};
    if constexpr (kMulti<F>) ba.mp = mpc;
    rc = dispatch_block<F>(MMAX, fld, ba, st, std::make_integer_sequence<int, FTraits<F>::MMAX + 1>{});
    if (rc) return rc;
    ColKArgs<F> ia;
    static_cast<ColArgs<F>&>(ia) = ColArgs<F>{ap, nullptr, ci, nullptr, n >> K, n, 0, 0, twf, twi, lsi, lk, io};
    if constexpr (kMulti<F>) ia.mp = mpc;
    rc = dispatch_cols<F, true>(K, fld, ia, cc, st, std::make_integer_sequence<int, KMAX>{});
    if (rc) return rc;
  }
  return FCIRC_OK;
}

}  // namespace fcirc

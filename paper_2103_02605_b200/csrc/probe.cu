// probe.cu — fcirc_primitive_rate: the measured integer throughput of the product's OWN ring
// primitives (R_const / R_var "measured modmul/s of K0's own const-twiddle and
// var x var primitives, in a register-resident all-SM microbenchmark"), used by bench.py as the
// roofline's integer peak, plus the raw IMAD.WIDE.U32 rate the multiplier-only ceiling is derived
// from.
//
// Every kind runs on all SMs at full occupancy (grid = SMs x resident CTAs of 256 threads), each
// thread carrying NCH independent dependency chains of the primitive in registers for `iters`
// iterations; operands come from the thread index so nothing is constant-folded, and the XOR of
// the chains is stored so nothing is dead.  The rate is primitives per second over one timed
// launch (CUDA events on the caller's stream) after one untimed warm-up launch.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/fcirc.h"
#include "modarith.cuh"
#include "runtime.h"

namespace fcirc {

constexpr int kProbeThreads = 256;
constexpr int NCH = 8;   // independent chains per thread

__device__ __forceinline__ uint64_t probe_seed(int c) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  return (t * 0x9E3779B97F4A7C15ull + (uint64_t)c * 0xD1B54A32D192ED03ull) % FieldGold::P;
}

template <int KIND>
__global__ void __launch_bounds__(kProbeThreads) k_probe(int64_t iters, uint64_t* sink) {
  uint64_t acc = 0;
  if constexpr (KIND == FCIRC_PRIM_GOLD_MUL || KIND == FCIRC_PRIM_GOLD_MULM || KIND == FCIRC_PRIM_GOLD_LEAF || KIND == FCIRC_PRIM_GOLD_FWD_A || KIND == FCIRC_PRIM_GOLD_FWD_B ||
                KIND == FCIRC_PRIM_GOLD_INV) {
    const FieldGold fld;
    uint64_t x[NCH], y[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) { x[c] = probe_seed(c); y[c] = probe_seed(c + NCH); }
    // constants < p (mulm's precondition): at most p - 2, odd
    const uint64_t s = (probe_seed(99) % (FieldGold::P - 2)) | 1, s2 = (probe_seed(98) % (FieldGold::P - 2)) | 1;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if constexpr (KIND == FCIRC_PRIM_GOLD_MUL) x[c] = FieldGold::mul(x[c], (c & 1) ? s : s2);
        else if constexpr (KIND == FCIRC_PRIM_GOLD_MULM) x[c] = FieldGold::mulm(x[c], (c & 1) ? s : s2);
        else if constexpr (KIND == FCIRC_PRIM_GOLD_LEAF) x[c] = fld.leaf(x[c], y[c]);
        else if constexpr (KIND == FCIRC_PRIM_GOLD_FWD_A) fld.fwd_a(x[c], y[c], (c & 1) ? s : s2);
        else if constexpr (KIND == FCIRC_PRIM_GOLD_FWD_B) fld.fwd_b(x[c], y[c], (c & 1) ? s : s2);
        else fld.inv(x[c], y[c], (c & 1) ? s : s2);
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc ^= x[c] ^ y[c];
  } else if constexpr (KIND == FCIRC_PRIM_U32_MULC || KIND == FCIRC_PRIM_U32_LEAF || KIND == FCIRC_PRIM_U32_FWD_A) {
    FieldU32 fld;
    fld.p = 998244353u;
    fld.p2 = 2u * fld.p;
    fld.pinv_neg = 998244351u;   // -p^-1 mod 2^32 for p = 998244353
    const TwU32 tw{(uint32_t)(probe_seed(99) % fld.p), 0};
    const TwU32 t2{tw.w, (uint32_t)(((uint64_t)tw.w << 32) / fld.p)};
    uint32_t x[NCH], y[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) { x[c] = (uint32_t)(probe_seed(c) % fld.p); y[c] = (uint32_t)(probe_seed(c + NCH) % fld.p); }
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if constexpr (KIND == FCIRC_PRIM_U32_MULC) x[c] = fld.mulc(x[c], t2);
        else if constexpr (KIND == FCIRC_PRIM_U32_LEAF) x[c] = fld.leaf(x[c], y[c]);
        else fld.fwd_a(x[c], y[c], t2);
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc ^= x[c] ^ y[c];
  } else if constexpr (KIND == FCIRC_PRIM_M31X2_MUL) {   // the paper's ring Z/(2^31-1)[sqrt 3]
    uint64_t x[NCH];
    const uint64_t s = (probe_seed(99) & 0x7FFFFFFE7FFFFFFEull);
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = probe_seed(c) & 0x7FFFFFFE7FFFFFFEull;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) x[c] = FieldM31x2::mul(x[c], s);
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc ^= x[c];
  } else {   // FCIRC_PRIM_IMAD_WIDE: raw 32 x 32 -> 64 products (the multiplier-only ceiling)
    // IMAD.WIDE.U32 with a zero addend, its two halves folded by one LOP3 on the ALU pipe (which runs
    // beside the FMA pipe): the highest IMAD.WIDE issue rate, so the strictest ceiling (an addend
    // register pair costs issue bandwidth: 25 instead of 31 per clock per SM measured)
    uint32_t x[NCH];
    const uint32_t m = (uint32_t)probe_seed(7) | 1u;
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = (uint32_t)probe_seed(c);
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t lo, hi;
        asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
                     : "=r"(lo), "=r"(hi) : "r"(x[c]), "r"(m));
        x[c] = lo ^ hi;
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc ^= x[c];
  }
  if (acc == 0x5bd1e995ull) sink[0] = acc;   // practically never: keeps the chains live
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[1] = acc;
}

// primitives per chain iteration (a butterfly counts one modmul: its twiddle product)
template <int KIND>
static int probe_run(int64_t iters, double* ops_per_s, double* ms, cudaStream_t st) {
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FCIRC_ECUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return FCIRC_ECUDA;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_probe<KIND>, kProbeThreads, 0) != cudaSuccess || occ < 1)
    return FCIRC_ECUDA;
  void* sink = nullptr;
  if (ws_alloc(dev, st, 16, &sink)) return FCIRC_ENOMEM;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned grid = (unsigned)(sms * occ);
  k_probe<KIND><<<grid, kProbeThreads, 0, st>>>(iters / 8 + 1, (uint64_t*)sink);   // warm-up
  cudaEventRecord(e0, st);
  k_probe<KIND><<<grid, kProbeThreads, 0, st>>>(iters, (uint64_t*)sink);
  cudaEventRecord(e1, st);
  int rc = cudaEventSynchronize(e1) == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
  float t = 0.f;
  if (rc == FCIRC_OK && cudaEventElapsedTime(&t, e0, e1) != cudaSuccess) rc = FCIRC_ECUDA;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ws_free(sink, st);
  if (rc) return rc;
  if (ms) *ms = t;
  if (ops_per_s) *ops_per_s = (double)grid * kProbeThreads * NCH * (double)iters / (t * 1e-3);
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

}  // namespace fcirc

extern "C" int fcirc_primitive_rate(int kind, int64_t iters, double* ops_per_s, double* ms, void* stream) {
  using namespace fcirc;
  if (iters < 1 || !ops_per_s) return FCIRC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  switch (kind) {
    case FCIRC_PRIM_GOLD_MUL: return probe_run<FCIRC_PRIM_GOLD_MUL>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_GOLD_FWD_A: return probe_run<FCIRC_PRIM_GOLD_FWD_A>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_GOLD_FWD_B: return probe_run<FCIRC_PRIM_GOLD_FWD_B>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_GOLD_INV: return probe_run<FCIRC_PRIM_GOLD_INV>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_U32_MULC: return probe_run<FCIRC_PRIM_U32_MULC>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_U32_LEAF: return probe_run<FCIRC_PRIM_U32_LEAF>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_U32_FWD_A: return probe_run<FCIRC_PRIM_U32_FWD_A>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_IMAD_WIDE: return probe_run<FCIRC_PRIM_IMAD_WIDE>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_M31X2_MUL: return probe_run<FCIRC_PRIM_M31X2_MUL>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_GOLD_MULM: return probe_run<FCIRC_PRIM_GOLD_MULM>(iters, ops_per_s, ms, st);
    case FCIRC_PRIM_GOLD_LEAF: return probe_run<FCIRC_PRIM_GOLD_LEAF>(iters, ops_per_s, ms, st);
    default: return FCIRC_EINVAL;
  }
}

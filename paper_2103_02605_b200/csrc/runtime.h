// runtime.h — internal (non-ABI) interface between the C-ABI layer (api.cu) and the per-field
// executors of the f-circulant product (matvec_u32.cu, matvec_gold.cu).  Splitting the fields
// into their own translation units lets the build compile them in parallel.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "modarith.cuh"
#include "plan.h"

namespace fcirc {

// A device-resident plan: the host tables of plan.h uploaded in the element layout of the field.
// Lifetime (api.cu): the tables are allocated stream-ordered on a private per-device stream and
// uploaded before the plan is published; every call that launches with the plan records an event
// on its stream (`uses`, one event per stream), and the destructor -- run when the plan cache has
// evicted the plan and the last caller holding it has finished enqueueing -- frees the tables with
// cudaFreeAsync on the private stream after waiting on those events: no device-wide
// synchronisation, no free before in-flight work is done.  Plans used inside a CUDA-graph capture
// are pinned by the cache (never evicted) because a graph may replay them at any later time.
struct DevPlan {
  HostPlan hp;
  int dev = 0;
  void* twf = nullptr;  // TwU32[n] or uint64_t[n]: s_{d,e} at heap index 2^d + e
  void* twi = nullptr;  // s_{d,e}^-1
  TwU32 last_si32{}, last_k32{};
  uint64_t last_si64 = 0, last_k64 = 0;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;   // guarded by the plan-cache mutex
  ~DevPlan();
};

// Opt-in dynamic shared memory above 48 KB for `fn` on the CURRENT device, once per (kernel, device)
// (kernel attributes are per device context): `mask` is one static per kernel instantiation.
inline bool smem_optin(const void* fn, size_t smem, std::atomic<uint32_t>& mask) {
  if (smem <= 48 * 1024) return true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const uint32_t bit = 1u << (dev & 31);
  if (mask.load(std::memory_order_acquire) & bit) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return true;
}

// integer tuning knob read once from the environment (FCIRC_<name>), else `dflt` (api.cu)
int knob(const char* name, int dflt);

// Launch a kernel of the path on `st`, with the programmatic-dependent-launch attribute when
// FCIRC_PDL (default 1; the kernels call pdl_entry(), modarith.cuh).
template <class... KArgs, class... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  static const int pdl = knob("PDL", 1);   // profiles/r02n_ab_pdl.txt: +0.3..4 %, default on
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch bookkeeping (api.cu): optional per-launch CUDA-event timing and the launch counter
void prof_begin(int kind, cudaStream_t st);
void prof_end(cudaStream_t st);
void count_launch();

// stream-ordered device scratch from the default memory pool (api.cu); free with ws_free on the same stream
int ws_alloc(int dev, cudaStream_t st, size_t bytes, void** out);
void ws_free(void* p, cudaStream_t st);

// bytes of a' + b' intermediates per chunk of the multi-pass schedule (FCIRC_CHUNK_BYTES)
size_t chunk_bytes();

// Per-field executors: all launches of one batched product on `st`.
// a, b, c: device arrays laid out as io describes; c may not alias a or b.
// io: EMB_PLAIN for fcirc_matvec; the applications pass their embedding (fcirc_kernels.cuh EmbedIO).
struct EmbedIO;
struct MultiPrime;
int run_matvec_u32(const FieldU32& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                   int64_t batch, cudaStream_t st, int dev, const EmbedIO& io);
// several 32-bit primes in one launch per pass (fcirc_kernels.cuh MultiPrime): batch = mp.n * mp.per
int run_matvec_u32m(const DevPlan& dp, const void* a, const void* b, void* c, int L, int64_t batch,
                    cudaStream_t st, int dev, const EmbedIO& io, const MultiPrime& mp);
int run_matvec_gold(const FieldGold& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                    int64_t batch, cudaStream_t st, int dev, const EmbedIO& io);
int run_matvec_m31(const FieldM31x2& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                   int64_t batch, cudaStream_t st, int dev, const EmbedIO& io);

// largest supported log2 n of the executors (multi-pass: sub-problem size + KMAX); kind = FieldKind
int max_log_n(int kind);
// log2 of the on-chip sub-problem size for n = 2^L (L <= split: one fused pass; else sub-problems)
int split_log_n(int kind, int L);
int split_log_n_u32(int L);
int split_log_n_m31(int L);

}  // namespace fcirc

// api.cu — libfcirc C ABI (include/fcirc.h): validation, plan cache, workspace, dispatch to the
// per-field executors (matvec_u32.cu, matvec_gold.cu; pass schedule in matvec_impl.cuh) and the
// applications (apps.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fcirc.h"
#include "apps.cuh"
#include "fcirc_kernels.cuh"
#include "plan.h"
#include "runtime.h"

namespace fcirc {

static thread_local int64_t g_launches = 0;

// NVTX ranges (SURVEY §5 tracing): one range per C-ABI call and, while kernel profiling is enabled,
// one per kernel launch (named by kind), so nsys / ncu --nvtx timelines show the pass structure.
// Header-only NVTX v3: a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
static const char* const kKindName[] = {"k_block fused", "k_block sub-problems", "k_cols forward", "k_cols inverse",
                                        "application kernels"};

// ------------------------------------------------------------------------------------------
// optional per-launch event timing (fcirc_profile_enable / fcirc_profile_read)
// ------------------------------------------------------------------------------------------
struct ProfRec { int kind; cudaEvent_t e0, e1; };
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_prof_pool;
static thread_local int t_prof_kind = -1;
static thread_local cudaEvent_t t_prof_e0 = nullptr;

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) { cudaEvent_t e = g_prof_pool.back(); g_prof_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_begin(int kind, cudaStream_t st) {
  if (!g_prof_on) return;
  nvtxRangePushA(kind >= 0 && kind < 5 ? kKindName[kind] : "kernel");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  t_prof_kind = kind;
  t_prof_e0 = prof_event();
  cudaEventRecord(t_prof_e0, st);
}
void prof_end(cudaStream_t st) {
  if (!g_prof_on || t_prof_kind < 0) return;
  nvtxRangePop();
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t e1 = prof_event();
  cudaEventRecord(e1, st);
  g_prof_recs.push_back({t_prof_kind, t_prof_e0, e1});
  t_prof_kind = -1;
}

// ------------------------------------------------------------------------------------------
// device plans
// ------------------------------------------------------------------------------------------
void count_launch() { ++g_launches; }

// Private per-device stream for plan uploads and stream-ordered table frees (non-blocking: never
// synchronises with the legacy default stream or with callers' streams).
static std::mutex g_priv_mu;
static std::map<int, cudaStream_t> g_priv;
static cudaStream_t plan_stream(int dev) {
  std::lock_guard<std::mutex> lk(g_priv_mu);
  auto it = g_priv.find(dev);
  if (it != g_priv.end()) return it->second;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  g_priv[dev] = s;
  return s;
}

DevPlan::~DevPlan() {
  // Runs when the cache has dropped the plan and the last caller holding it has enqueued its work
  // (and recorded its use event).  Frees stream-ordered after every recorded use: no device sync.
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaStream_t ps = plan_stream(dev);
  for (auto& u : uses) {
    if (ps) cudaStreamWaitEvent(ps, u.second, 0);
    cudaEventDestroy(u.second);   // released by the driver once the event has completed
  }
  if (twf) cudaFreeAsync(twf, ps);
  if (twi) cudaFreeAsync(twi, ps);
  if (cur != dev) cudaSetDevice(cur);
}

static std::mutex g_mu;
static std::mutex g_host_mu;
// plan cache keyed by (device, p, f, log2 n), least-recently-used eviction beyond kMaxPlans entries or
// kMaxPlanBytes of device tables (callers with a new f per call would otherwise grow it without
// bound).  Evicted tables are freed by DevPlan::~DevPlan after their recorded uses (stream-ordered).
// A plan used while its stream is capturing a CUDA graph is pinned: never evicted (a graph may
// replay it any time later); only fcirc_release_cache drops pinned plans.
struct PlanEntry {
  std::shared_ptr<DevPlan> plan;
  uint64_t last_use = 0;
  size_t bytes = 0;
  bool pinned = false;
};
static std::map<std::tuple<int, uint64_t, uint64_t, int>, PlanEntry> g_plans;
static uint64_t g_plan_tick = 0;
static size_t g_plan_bytes = 0;
static constexpr size_t kMaxPlans = 64;
static constexpr size_t kMaxPlanBytes = (size_t)2 << 30;

static void evict_plans_locked() {
  for (;;) {
    size_t unpinned = 0;
    for (auto& kv : g_plans) unpinned += !kv.second.pinned;
    if (!(unpinned > 0 && (g_plans.size() > kMaxPlans || (g_plan_bytes > kMaxPlanBytes && g_plans.size() > 1))))
      return;
    auto victim = g_plans.end();
    for (auto it = g_plans.begin(); it != g_plans.end(); ++it)
      if (!it->second.pinned && (victim == g_plans.end() || it->second.last_use < victim->second.last_use)) victim = it;
    if (victim == g_plans.end() || g_plans.size() - 1 < 1) return;
    g_plan_bytes -= victim->second.bytes;
    g_plans.erase(victim);
  }
}

// After a call enqueued work that reads the plan's tables on `st`: record (or re-record) the plan's
// use event for `st`.  (Under capture get_plan has pinned the plan instead.)
static void note_plan_use(DevPlan* dp, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t ev = nullptr;
  for (auto& u : dp->uses)
    if (u.first == st) ev = u.second;
  if (!ev) {
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;
    dp->uses.emplace_back(st, ev);
  }
  cudaEventRecord(ev, st);
}

static TwU32 shoup_pair(uint64_t w, uint64_t p) {
  TwU32 t;
  t.w = (uint32_t)w;
  t.q = (uint32_t)((((unsigned __int128)w) << 32) / p);
  return t;
}

// allocate + upload one table on the private stream (completion is awaited before publication)
static int upload(void** dst, const void* src, size_t bytes, cudaStream_t ps) {
  if (cudaMallocAsync(dst, bytes, ps) != cudaSuccess) return FCIRC_ENOMEM;
  return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, ps) == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

static int get_plan(int dev, uint64_t p, uint64_t f, int L, cudaStream_t st, std::shared_ptr<DevPlan>* out) {
  auto key = std::make_tuple(dev, p, f, L);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      it->second.last_use = ++g_plan_tick;
      if (capturing) it->second.pinned = true;   // a captured graph may replay it at any later time
      *out = it->second.plan;
      return FCIRC_OK;
    }
  }
  // a new plan needs host work, allocations and a synchronous upload: not inside a graph capture
  if (capturing) return FCIRC_EINVAL;
  auto dp = std::make_shared<DevPlan>();
  dp->dev = dev;
  int st_ = build_host_plan(p, f, L, &dp->hp);
  if (st_ != FCIRC_OK) return st_;
  cudaStream_t ps = plan_stream(dev);
  if (!ps) return FCIRC_ECUDA;
  const PrimeInfo* pi = prime_info(p);
  const size_t n = dp->hp.s.size();
  size_t bytes = 0;
  int rc = FCIRC_OK;
  std::vector<TwU32> hf, hi;
  std::vector<uint64_t> mf, mi;   // (host staging stays alive until the synchronisation below)
  if (!pi->wide) {
    hf.resize(n);
    hi.resize(n);
    for (size_t i = 0; i < n; ++i) { hf[i] = shoup_pair(dp->hp.s[i], p); hi[i] = shoup_pair(dp->hp.sinv[i], p); }
    bytes = 2 * n * sizeof(TwU32);
    if (!rc) rc = upload(&dp->twf, hf.data(), n * sizeof(TwU32), ps);
    if (!rc) rc = upload(&dp->twi, hi.data(), n * sizeof(TwU32), ps);
    dp->last_si32 = shoup_pair(dp->hp.last_si, p);
    dp->last_k32 = shoup_pair(dp->hp.K, p);
  } else if (pi->kind == KIND_GOLD) {
    // Montgomery form of every constant operand (FieldGold::mulm): s R mod p with R = 2^64,
    // 2^64 mod p = 2^32 - 1.  The host plan (fcirc_plan_table) keeps the plain values.
    const uint64_t R = 0xFFFFFFFFull;
    mf.resize(n);
    mi.resize(n);
    for (size_t i = 0; i < n; ++i) { mf[i] = mulmod(dp->hp.s[i], R, p); mi[i] = mulmod(dp->hp.sinv[i], R, p); }
    bytes = 2 * n * 8;
    if (!rc) rc = upload(&dp->twf, mf.data(), n * 8, ps);
    if (!rc) rc = upload(&dp->twi, mi.data(), n * 8, ps);
    // the leaves are Montgomery products too (a b R^-1): the final scaling undoes that R
    const uint64_t R2 = mulmod(R, R, p);
    dp->last_si64 = mulmod(dp->hp.last_si, R2, p);
    dp->last_k64 = mulmod(dp->hp.K, R2, p);
  } else {
    bytes = 2 * n * 8;
    if (!rc) rc = upload(&dp->twf, dp->hp.s.data(), n * 8, ps);
    if (!rc) rc = upload(&dp->twi, dp->hp.sinv.data(), n * 8, ps);
    dp->last_si64 = dp->hp.last_si;
    dp->last_k64 = dp->hp.K;
  }
  // the tables are complete on the device before any caller's stream can use the plan
  if (cudaStreamSynchronize(ps) != cudaSuccess && !rc) rc = FCIRC_ECUDA;
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {  // another thread won
    it->second.last_use = ++g_plan_tick;
    *out = it->second.plan;
    return FCIRC_OK;
  }
  g_plans[key] = PlanEntry{dp, ++g_plan_tick, bytes, false};
  g_plan_bytes += bytes;
  evict_plans_locked();
  *out = dp;
  return FCIRC_OK;
}

// ------------------------------------------------------------------------------------------
// workspace: stream-ordered allocations from the device's default memory pool (cudaMallocAsync /
// cudaFreeAsync on the call's stream).  The pool keeps freed blocks (release threshold raised to
// the maximum), so after the first call this costs no cudaMalloc; calls on different streams never
// share scratch; and the allocations are capturable, so a whole product can be recorded in a CUDA
// graph (bench.py --graph).
// ------------------------------------------------------------------------------------------
int ws_alloc(int dev, cudaStream_t st, size_t bytes, void** out) {
  static std::mutex mu;
  static std::map<int, bool> configured;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!configured[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      configured[dev] = true;
    }
  }
  if (cudaMallocAsync(out, bytes, st) != cudaSuccess) return FCIRC_ENOMEM;
  return FCIRC_OK;
}

void ws_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

size_t chunk_bytes() {
  static size_t v = [] {
    const char* e = getenv("FCIRC_CHUNK_BYTES");
    return e ? (size_t)strtoull(e, nullptr, 10) : (size_t)1 << 30;  // profiles/r01c_sweep.txt
  }();
  return v;
}

int knob(const char* name, int dflt) {
  char key[64];
  snprintf(key, sizeof key, "FCIRC_%s", name);
  const char* e = getenv(key);
  return e ? atoi(e) : dflt;
}

static FieldU32 make_u32(uint64_t p) {
  FieldU32 fld;
  fld.p = (uint32_t)p;
  fld.p2 = (uint32_t)(2 * p);
  uint32_t inv = 1;  // p^-1 mod 2^32 by Newton iteration (5 steps: 1 -> 32 correct bits)
  for (int i = 0; i < 5; ++i) inv *= 2u - (uint32_t)p * inv;
  fld.pinv_neg = (uint32_t)(0u - inv);
  return fld;
}

static bool overlaps(const void* x, size_t xb, const void* y, size_t yb) {
  const char* a0 = (const char*)x; const char* b0 = (const char*)y;
  return a0 < b0 + yb && b0 < a0 + xb;
}

static int ilog2_exact(int64_t n) {
  if (n < 1 || (n & (n - 1))) return -1;
  int L = 0;
  while (((int64_t)1 << L) < n) ++L;
  return L;
}

// ------------------------------------------------------------------------------------------
// optional input validation (FCIRC_CHECK_INPUTS=1): inputs must be canonical residues (< p); the
// product path does not check this on the device.  In checking mode a counting kernel runs first
// and the call synchronises the stream and returns FCIRC_EINVAL if any element is >= p.
// ------------------------------------------------------------------------------------------
template <class E, bool PACKED>
__global__ void k_count_noncanonical(const E* __restrict__ x, int64_t count, uint64_t p,
                                     unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = (uint64_t)x[i];
    local += PACKED ? ((v & 0xFFFFFFFFull) >= p || (v >> 32) >= p) : v >= p;
  }
  if (local) atomicAdd(bad, local);
}

static int check_canonical(uint64_t p, const PrimeInfo* pi, const void* x, int64_t count, cudaStream_t st) {
  static const bool on = knob("CHECK_INPUTS", 0) != 0;
  if (!on || count <= 0) return FCIRC_OK;
  unsigned long long* d = nullptr;
  unsigned long long h = 0;
  if (cudaMallocAsync((void**)&d, sizeof h, st) != cudaSuccess) return FCIRC_ENOMEM;
  cudaMemsetAsync(d, 0, sizeof h, st);
  const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 148 * 8);
  if (pi->kind == KIND_M31X2) k_count_noncanonical<uint64_t, true><<<blocks, 256, 0, st>>>((const uint64_t*)x, count, p, d);
  else if (pi->wide) k_count_noncanonical<uint64_t, false><<<blocks, 256, 0, st>>>((const uint64_t*)x, count, p, d);
  else k_count_noncanonical<uint32_t, false><<<blocks, 256, 0, st>>>((const uint32_t*)x, count, p, d);
  cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return FCIRC_ECUDA;
  return h ? FCIRC_EINVAL : FCIRC_OK;
}

// plan lookup + dispatch of one batched product (no argument validation; callers validate)
static int matvec_core(uint64_t p, uint64_t f, const void* a, const void* b, void* c, int L, int64_t batch,
                       cudaStream_t st, const EmbedIO& io) {
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  if (L > pi->two_adicity || L > max_log_n(pi->kind)) return FCIRC_ESIZE;
  if (pi->kind != KIND_M31X2) f %= p;   // packed Z/p[sqrt 3] scalars are validated, not reduced
  // Theorem 1 premises checked on the host before touching the device
  int rc = check_premises(pi, f, L);
  if (rc) return rc;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FCIRC_ECUDA;
  std::shared_ptr<DevPlan> dp;
  rc = get_plan(dev, p, f, L, st, &dp);
  if (rc) return rc;
  if (pi->kind == KIND_GOLD) {
    FieldGold fld;
    rc = run_matvec_gold(fld, *dp, a, b, c, L, batch, st, dev, io);
  } else if (pi->kind == KIND_M31X2) {
    FieldM31x2 fld;
    rc = run_matvec_m31(fld, *dp, a, b, c, L, batch, st, dev, io);
  } else {
    rc = run_matvec_u32(make_u32(p), *dp, a, b, c, L, batch, st, dev, io);
  }
  note_plan_use(dp.get(), st);   // even after a failed launch: some kernels may be queued
  return rc;
}

// fcirc_matvec without resetting the launch counter (also used by the host pipeline)
static int matvec_impl(uint64_t p, uint64_t f, const void* a, const void* b, void* c, int64_t n, int64_t batch,
                       cudaStream_t st) {
  if (!a || !b || !c || n < 1 || batch < 1) return FCIRC_EINVAL;
  const int L = ilog2_exact(n);
  if (L < 0) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  const size_t es = pi->wide ? 8 : 4;
  if (L > pi->two_adicity || L > max_log_n(pi->kind)) return FCIRC_ESIZE;
  const size_t bytes = (size_t)n * (size_t)batch * es;
  if (overlaps(c, bytes, a, bytes) || overlaps(c, bytes, b, bytes)) return FCIRC_EINVAL;
  int rc = check_canonical(p, pi, a, n * batch, st);
  if (rc == FCIRC_OK) rc = check_canonical(p, pi, b, n * batch, st);
  if (rc) return rc;
  return matvec_core(p, f, a, b, c, L, batch, st, EmbedIO{});
}

static int64_t next_pow2(int64_t x) {
  int64_t r = 1;
  while (r < x) r <<= 1;
  return r;
}

// polynomial product through an f = 1 circulant of order L (reading R8): the
// a~ embedding is fused into the first pass's loads and the truncation into the last pass's stores
static int polymul_impl(uint64_t p, const void* a, int64_t na, const void* b, int64_t nb, void* c, int64_t batch,
                        cudaStream_t st) {
  EmbedIO io;
  io.mode = EMB_POLY;
  io.na = na;
  io.nb = nb;
  io.nc = na + nb - 1;
  return matvec_core(p, 1, a, b, c, ilog2_exact(next_pow2(io.nc)), batch, st, io);
}

// host buffers -> device -> host, pipelined over NSLOT streams (fcirc_matvec_host).  Each call takes
// a context (streams + device staging buffers) from a per-device pool and returns it afterwards, so
// concurrent host threads run their pipelines concurrently (one mutex only around take / return).
struct HostCtx {
  static constexpr int NSLOT = 3;
  int dev = 0;
  cudaStream_t st[NSLOT] = {};
  void* buf[NSLOT] = {};
  size_t bytes = 0;
};
static std::vector<HostCtx*> g_host_free;   // idle contexts (any device), guarded by g_host_mu

static HostCtx* host_ctx_take(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_host_mu);
    for (size_t i = 0; i < g_host_free.size(); ++i)
      if (g_host_free[i]->dev == dev) {
        HostCtx* hc = g_host_free[i];
        g_host_free.erase(g_host_free.begin() + i);
        return hc;
      }
  }
  HostCtx* hc = new HostCtx;
  hc->dev = dev;
  for (int i = 0; i < HostCtx::NSLOT; ++i)
    if (cudaStreamCreateWithFlags(&hc->st[i], cudaStreamNonBlocking) != cudaSuccess) { delete hc; return nullptr; }
  return hc;
}
static void host_ctx_return(HostCtx* hc) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  g_host_free.push_back(hc);
}

static int host_pipeline(uint64_t p, uint64_t f, const char* a, const char* b, char* c, int64_t n, int64_t batch,
                         size_t es, int dev) {
  const size_t inst_bytes = (size_t)n * es;
  static const int64_t chunk_mb = std::max(1, knob("HOST_CHUNK_MB", 32));  // per operand and chunk
  const int64_t C = std::max<int64_t>(1, std::min<int64_t>(batch, (chunk_mb << 20) / (int64_t)inst_bytes));
  const size_t slot_bytes = 3 * (size_t)C * inst_bytes;
  HostCtx* hc = host_ctx_take(dev);
  if (!hc) return FCIRC_ECUDA;
  struct Ret { HostCtx* h; ~Ret() { host_ctx_return(h); } } ret{hc};
  if (hc->bytes < slot_bytes) {
    for (int i = 0; i < HostCtx::NSLOT; ++i) {
      cudaStreamSynchronize(hc->st[i]);
      if (hc->buf[i]) cudaFreeAsync(hc->buf[i], hc->st[i]);
      hc->buf[i] = nullptr;
    }
    hc->bytes = 0;
    for (int i = 0; i < HostCtx::NSLOT; ++i)
      if (cudaMallocAsync(&hc->buf[i], slot_bytes, hc->st[i]) != cudaSuccess) return FCIRC_ENOMEM;
    hc->bytes = slot_bytes;
  }
  int rc = FCIRC_OK;
  int64_t chunk = 0;
  for (int64_t i0 = 0; i0 < batch && rc == FCIRC_OK; i0 += C, ++chunk) {
    const int64_t cc = std::min<int64_t>(C, batch - i0);
    const int sl = (int)(chunk % HostCtx::NSLOT);
    cudaStream_t st = hc->st[sl];
    char* dA = (char*)hc->buf[sl];
    char* dB = dA + (size_t)C * inst_bytes;
    char* dC = dB + (size_t)C * inst_bytes;
    const size_t off = (size_t)i0 * inst_bytes, nb = (size_t)cc * inst_bytes;
    if (cudaMemcpyAsync(dA, a + off, nb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(dB, b + off, nb, cudaMemcpyHostToDevice, st) != cudaSuccess) { rc = FCIRC_ECUDA; break; }
    rc = matvec_impl(p, f, dA, dB, dC, n, cc, st);
    if (rc) break;
    if (cudaMemcpyAsync(c + off, dC, nb, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = FCIRC_ECUDA;
  }
  for (int i = 0; i < HostCtx::NSLOT; ++i)
    if (cudaStreamSynchronize(hc->st[i]) != cudaSuccess && rc == FCIRC_OK) rc = FCIRC_ECUDA;
  return rc;
}

// big-integer product (reading R12)
static int bigint_impl(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z, int64_t batch,
                       cudaStream_t st) {
  const uint64_t P1 = 998244353ull, P2 = 469762049ull, P3 = 167772161ull;
  const int64_t nd = 2 * (nx + ny), ncoef = nd - 1;
  const int64_t L = next_pow2(ncoef);
  if (ilog2_exact(L) > 23) return FCIRC_ESIZE;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FCIRC_ECUDA;
  const int64_t nseg = (nd + kCarrySeg - 1) / kCarrySeg;
  const size_t need = (size_t)(3 * batch * L) * 4 + (size_t)(batch * nd) * 4 + (size_t)(batch * nseg) * 4;
  void* ws;
  int rc = ws_alloc(dev, st, need, &ws);
  if (rc) return rc;
  struct Free { void* p; cudaStream_t s; ~Free() { ws_free(p, s); } } free_ws{ws, st};
  uint32_t* r1 = (uint32_t*)ws;
  uint32_t* r2 = r1 + batch * L;
  uint32_t* r3 = r2 + batch * L;
  uint32_t* E = r3 + batch * L;
  uint32_t* S = E + batch * nd;
  // 16-bit limb split + a~ embedding fused into the first pass (EMB_LIMBS); the three primes' f = 1
  // products run as ONE product of 3 batch instances per pass (instance q batch + i = prime q,
  // operands of instance i), outputs r1 | r2 | r3 contiguous.  FCIRC_BIGINT_SPLIT=1
  // issues the three products separately (A/B).
  EmbedIO io;
  io.mode = EMB_LIMBS;
  io.na = nx;
  io.nb = ny;
  const int lg = ilog2_exact(L);
  static const int split = knob("BIGINT_SPLIT", 0);
  if (split) {
    if ((rc = matvec_core(P1, 1, x, y, r1, lg, batch, st, io))) return rc;
    if ((rc = matvec_core(P2, 1, x, y, r2, lg, batch, st, io))) return rc;
    if ((rc = matvec_core(P3, 1, x, y, r3, lg, batch, st, io))) return rc;
  } else {
    const uint64_t ps[3] = {P1, P2, P3};
    std::shared_ptr<DevPlan> dp[3];
    MultiPrime mp;
    mp.n = 3;
    mp.per = batch;
    for (int q = 0; q < 3; ++q) {
      if ((rc = get_plan(dev, ps[q], 1, lg, st, &dp[q]))) return rc;
      mp.ps[q] = PrimeSel{make_u32(ps[q]), (const TwU32*)dp[q]->twf, (const TwU32*)dp[q]->twi, dp[q]->last_si32,
                          dp[q]->last_k32};
    }
    rc = run_matvec_u32m(*dp[0], x, y, r1, lg, 3 * batch, st, dev, io, mp);
    for (int q = 0; q < 3; ++q) note_plan_use(dp[q].get(), st);
    if (rc) return rc;
  }
  GarnerConsts g;
  g.p1 = (uint32_t)P1; g.p2 = (uint32_t)P2; g.p3 = (uint32_t)P3;
  g.p1p2 = P1 * P2;
  g.one2q = (uint32_t)((1ull << 32) / P2);
  g.one3q = (uint32_t)((1ull << 32) / P3);
  g.c12 = (uint32_t)invmod(P1 % P2, P2);
  g.c12q = (uint32_t)(((uint64_t)g.c12 << 32) / P2);
  g.p1m3 = (uint32_t)(P1 % P3);
  g.p1m3q = (uint32_t)(((uint64_t)g.p1m3 << 32) / P3);
  g.c123 = (uint32_t)invmod(mulmod(P1 % P3, P2 % P3, P3), P3);
  g.c123q = (uint32_t)(((uint64_t)g.c123 << 32) / P3);
  prof_begin(4, st);
  launch_k(k_crt_digits, (unsigned)(batch * nseg), kCarryThreads, 0, st, (const uint32_t*)r1, (const uint32_t*)r2,
           (const uint32_t*)r3, (int64_t)L, (int64_t)ncoef, (int64_t)nd, (int64_t)nseg, g, E, S);
  prof_end(st);
  prof_begin(4, st);
  launch_k(k_carry_top, (unsigned)batch, kTopThreads, 0, st, S, (int64_t)nseg);
  prof_end(st);
  prof_begin(4, st);
  launch_k(k_carry_apply, (unsigned)(batch * nseg), kCarryThreads, 0, st, (const uint32_t*)E, (int64_t)nd, (int64_t)nseg,
           (const uint32_t*)S, z, (int64_t)(nx + ny));
  prof_end(st);
  g_launches += 3;   // k_crt_digits, k_carry_top, k_carry_apply
  return cudaPeekAtLastError() == cudaSuccess ? FCIRC_OK : FCIRC_ECUDA;
}

}  // namespace fcirc

using namespace fcirc;

extern "C" {

int bigint_mul(const uint32_t* x, int64_t nx, const uint32_t* y, int64_t ny, uint32_t* z, int64_t batch,
               void* stream) {
  NvtxRange nvtx_range("bigint_mul");
  g_launches = 0;
  if (!x || !y || !z || nx < 1 || ny < 1 || batch < 1) return FCIRC_EINVAL;
  if (overlaps(z, (size_t)((nx + ny) * batch) * 4, x, (size_t)(nx * batch) * 4) ||
      overlaps(z, (size_t)((nx + ny) * batch) * 4, y, (size_t)(ny * batch) * 4))
    return FCIRC_EINVAL;
  return bigint_impl(x, nx, y, ny, z, batch, (cudaStream_t)stream);
}

int fcirc_matvec(uint64_t p, uint64_t f, const void* a, const void* b, void* c, int64_t n, int64_t batch,
                 void* stream) {
  NvtxRange nvtx_range("fcirc_matvec");
  g_launches = 0;
  return matvec_impl(p, f, a, b, c, n, batch, (cudaStream_t)stream);
}

int fcirc_circulant_matvec(uint64_t p, const void* a, const void* b, void* c, int64_t n, int64_t batch,
                           void* stream) {
  NvtxRange nvtx_range("fcirc_circulant_matvec");
  g_launches = 0;
  if (!a || !b || !c || n < 1 || batch < 1) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  const size_t es = pi->wide ? 8 : 4;
  const size_t bytes = (size_t)n * (size_t)batch * es;
  if (overlaps(c, bytes, a, bytes) || overlaps(c, bytes, b, bytes)) return FCIRC_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = check_canonical(p, pi, a, n * batch, st);
  if (rc == FCIRC_OK) rc = check_canonical(p, pi, b, n * batch, st);
  if (rc) return rc;
  if ((n & (n - 1)) == 0) return matvec_core(p, 1, a, b, c, ilog2_exact(n), batch, st, EmbedIO{});
  // Corollary 1: order N = the smallest power of two >= 2n - 1 (reading R10)
  const int64_t N = next_pow2(2 * n - 1);
  const int LN = ilog2_exact(N);
  if (LN > pi->two_adicity || LN > max_log_n(pi->kind)) return FCIRC_ESIZE;
  EmbedIO io;
  io.mode = EMB_ANYN;
  io.na = n;
  io.nb = n;
  io.nc = n;
  return matvec_core(p, 1, a, b, c, LN, batch, st, io);
}

int fcirc_matvec_host(uint64_t p, uint64_t f, const void* a, const void* b, void* c, int64_t n,
                      int64_t batch) {
  NvtxRange nvtx_range("fcirc_matvec_host");
  g_launches = 0;
  if (!a || !b || !c || n < 1 || batch < 1) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  const int L = ilog2_exact(n);
  if (L < 0) return FCIRC_EINVAL;
  const size_t es = pi->wide ? 8 : 4;
  const size_t bytes = (size_t)n * (size_t)batch * es;
  if (overlaps(c, bytes, a, bytes) || overlaps(c, bytes, b, bytes)) return FCIRC_EINVAL;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FCIRC_ECUDA;
  return host_pipeline(p, f, (const char*)a, (const char*)b, (char*)c, n, batch, es, dev);
}

int fcirc_polymul(uint64_t p, const void* a, int64_t na, const void* b, int64_t nb, void* c, int64_t batch,
                  void* stream) {
  NvtxRange nvtx_range("fcirc_polymul");
  g_launches = 0;
  if (!a || !b || !c || na < 1 || nb < 1 || batch < 1) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  const size_t es = pi->wide ? 8 : 4;
  const int64_t nc = na + nb - 1;
  if (overlaps(c, (size_t)(nc * batch) * es, a, (size_t)(na * batch) * es) ||
      overlaps(c, (size_t)(nc * batch) * es, b, (size_t)(nb * batch) * es))
    return FCIRC_EINVAL;
  const int64_t L = next_pow2(nc);
  if (ilog2_exact(L) > pi->two_adicity || ilog2_exact(L) > max_log_n(pi->kind)) return FCIRC_ESIZE;
  int rc = check_canonical(p, pi, a, na * batch, (cudaStream_t)stream);
  if (rc == FCIRC_OK) rc = check_canonical(p, pi, b, nb * batch, (cudaStream_t)stream);
  if (rc) return rc;
  return polymul_impl(p, a, na, b, nb, c, batch, (cudaStream_t)stream);
}

const char* fcirc_strerror(int status) {
  switch (status) {
    case FCIRC_OK: return "ok";
    case FCIRC_EINVAL: return "invalid argument (null pointer, size < 1, n not a power of two, or overlap)";
    case FCIRC_EPRIME: return "modulus not in the registry";
    case FCIRC_ENOROOT: return "f is zero or has no n-th root mod p";
    case FCIRC_ESIZE: return "size unsupported: no n-th root of unity mod p, or above the maximum";
    case FCIRC_ENOMEM: return "device allocation failed";
    case FCIRC_ECUDA: return "CUDA error";
    default: return "unknown status";
  }
}

int fcirc_plan_table(uint64_t p, uint64_t f, int64_t n, uint64_t* s, uint64_t* sinv, uint64_t* w, uint64_t* K) {
  if (!s || !sinv || !w || !K) return FCIRC_EINVAL;
  const int L = ilog2_exact(n);
  if (L < 0) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  if (L > pi->two_adicity) return FCIRC_ESIZE;
  HostPlan hp;
  int rc = build_host_plan(p, f, L, &hp);
  if (rc) return rc;
  std::copy(hp.s.begin(), hp.s.end(), s);
  std::copy(hp.sinv.begin(), hp.sinv.end(), sinv);
  *w = hp.w;
  *K = hp.K;
  return FCIRC_OK;
}

const char* fcirc_version(void) { return "libfcirc 0.1 sm_100a"; }

int fcirc_schedule(uint64_t p, int64_t n, int* sub_log, int* top_levels) {
  if (!sub_log || !top_levels) return FCIRC_EINVAL;
  const int L = ilog2_exact(n);
  if (L < 0) return FCIRC_EINVAL;
  const PrimeInfo* pi = prime_info(p);
  if (!pi) return FCIRC_EPRIME;
  if (L > pi->two_adicity || L > max_log_n(pi->kind)) return FCIRC_ESIZE;
  const int S = split_log_n(pi->kind, L);
  *sub_log = L <= S ? L : S;
  *top_levels = L <= S ? 0 : L - S;
  return FCIRC_OK;
}

int64_t fcirc_last_launch_count(void) { return g_launches; }

int fcirc_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return FCIRC_OK;
}

int fcirc_profile_read(int64_t* counts, double* ms, int nkinds) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int i = 0; i < nkinds; ++i) { if (counts) counts[i] = 0; if (ms) ms[i] = 0.0; }
  int rc = FCIRC_NKINDS;
  for (auto& r : g_prof_recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&t, r.e0, r.e1) != cudaSuccess)
      rc = FCIRC_ECUDA;
    if (r.kind < nkinds) {
      if (counts) counts[r.kind] += 1;
      if (ms) ms[r.kind] += t;
    }
    g_prof_pool.push_back(r.e0);
    g_prof_pool.push_back(r.e1);
  }
  g_prof_recs.clear();
  return rc;
}

int fcirc_release_cache(void) {
  // drops every plan, pinned ones included: CUDA graphs captured over libfcirc calls must not be
  // replayed afterwards (fcirc.h)
  cudaDeviceSynchronize();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_plans.clear();
    g_plan_bytes = 0;
  }
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaStream_t ps = plan_stream(dev);
    if (ps) cudaStreamSynchronize(ps);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  return FCIRC_OK;
}

int64_t fcirc_plan_count(int* pinned) {
  std::lock_guard<std::mutex> lk(g_mu);
  int np = 0;
  for (auto& kv : g_plans) np += kv.second.pinned;
  if (pinned) *pinned = np;
  return (int64_t)g_plans.size();
}

}  // extern "C"

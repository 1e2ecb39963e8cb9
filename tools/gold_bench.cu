// tools/gold_bench.cu — throughput + correctness of Goldilocks butterfly variants (dev tool).
// Each variant runs register-resident butterfly chains on all SMs; results are checked against a
// slow __int128 reference computed on the device.  Output: JSON lines.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2103_02605_b200/csrc/modarith.cuh"

using namespace fcirc;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr uint64_t P = 0xFFFFFFFF00000001ull;
__device__ __forceinline__ uint64_t ref_mul(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * b) % P);
}
__device__ __forceinline__ uint64_t ref_add(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)(a % P) + (b % P)) % P);
}
__device__ __forceinline__ uint64_t ref_sub(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)(a % P) + P - (b % P)) % P);
}

constexpr int CH = 8, IT = 1024;

template <int KIND>
__global__ void __launch_bounds__(256) k_tp(uint64_t* out, uint64_t seed) {
  FieldGold F;
  uint64_t x[CH], y[CH];
  for (int c = 0; c < CH; ++c) { x[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B97F4A7C15ull; y[c] = x[c] ^ 0xDEADBEEFCAFEF00Dull; }
  const uint64_t w = 0x1234567890ABCDEFull ^ seed;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (KIND == 0) F.fwd_a(x[c], y[c], w);
      if (KIND == 1) F.fwd_b(x[c], y[c], w);
      if (KIND == 2) F.inv(x[c], y[c], w);
      if (KIND == 3) x[c] = F.mul(x[c], w);
    }
  }
  uint64_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ y[c];
  if (acc == 0x42) out[0] = acc;
}

// correctness: random and edge operands vs reference
__global__ void k_check(unsigned long long* bad, uint64_t seed) {
  FieldGold F;
  const uint64_t edge[] = {0, 1, 2, P - 1, P, P + 1, 0xFFFFFFFFFFFFFFFFull, 0xFFFFFFFF00000000ull,
                           0x00000000FFFFFFFFull, 0x8000000000000000ull, 0xFFFFFFFEFFFFFFFFull, P - 2};
  uint64_t s = seed ^ (threadIdx.x + blockIdx.x * 977ull);
  for (int i = 0; i < 256; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t a = s;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t b = s;
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t w = s % P;
    if (i < 144) { a = edge[i % 12]; b = edge[(i / 12) % 12]; }
    // mul: any inputs -> canonical result required by the product's invariants
    uint64_t m = F.mul(a, b);
    if (m != ref_mul(a, b)) atomicAdd(bad, 1ull);
    // forward a: weak inputs
    uint64_t x = a, y = b;
    F.fwd_a(x, y, w);
    uint64_t t = ref_mul(b, w);
    if (x % P != ref_add(a, t) || y % P != ref_sub(a, t)) atomicAdd(bad + 1, 1ull);
    x = a; y = b;
    F.fwd_b(x, y, w);
    t = ref_mul(a, w);
    if (x % P != ref_add(t, b) || y % P != ref_sub(t, b)) atomicAdd(bad + 2, 1ull);
    // inverse: canonical inputs (invariant of the inverse chain)
    uint64_t u = a % P, v = b % P;
    F.inv(u, v, w);
    if (u != ref_mul(ref_add(a, b), w) || v % P != ref_sub(a, b)) atomicAdd(bad + 3, 1ull);
    if (F.canon(a) != a % P) atomicAdd(bad + 4, 1ull);
  }
}

template <int KIND>
static int tp(const char* name, int nsm) {
  uint64_t* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int blocks = nsm * 4, thr = 256;
  k_tp<KIND><<<blocks, thr>>>(d, 1); CK(cudaDeviceSynchronize());
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0)); k_tp<KIND><<<blocks, thr>>>(d, r + 2); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  double ops = (double)blocks * thr * CH * IT;
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"variant\": \"%s\", \"ms\": %.4f, \"per_s\": %.4e, \"per_clk_sm_at_max\": %.3f}\n", name, best,
         ops / (best * 1e-3), ops / (best * 1e-3) / nsm / (clk * 1e3));
  return 0;
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* bad; CK(cudaMalloc(&bad, 5 * 8)); CK(cudaMemset(bad, 0, 5 * 8));
  k_check<<<148, 256>>>(bad, 12345); CK(cudaDeviceSynchronize());
  unsigned long long h[5]; CK(cudaMemcpy(h, bad, 40, cudaMemcpyDeviceToHost));
  printf("{\"check_bad\": [%llu, %llu, %llu, %llu, %llu]}\n", h[0], h[1], h[2], h[3], h[4]);
  tp<0>("fwd_a butterfly", nsm);
  tp<1>("fwd_b butterfly", nsm);
  tp<2>("inv butterfly", nsm);
  tp<3>("mul chain", nsm);
  return (h[0] | h[1] | h[2] | h[3] | h[4]) ? 2 : 0;
}

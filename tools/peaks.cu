// tools/peaks.cu — integer-pipe microbenchmarks for the libfcirc roofline.
//
// Measures, on all SMs with register-resident independent chains:
//   * raw instruction throughput: IMAD (lo), IMAD.HI, IMAD.WIDE.U32, IADD3, LOP3
//   * modmul throughput of the primitives the hot path uses:
//       shoup32  (const x var, twiddle + precomputed quotient),
//       mont32   (var x var Montgomery),
//       gold64   (Goldilocks 64x64 -> 128 -> special reduction)
// Reported per SM per clock (clock taken from clock64 deltas inside the kernel)
// and per second.  Output: one JSON object per line.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o peaks tools/peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 8;         // independent chains per thread
constexpr int ITERS = 4096;   // loop trips

__device__ unsigned long long g_clk[2048];

template <int OP>
__global__ void __launch_bounds__(512) k_raw(uint32_t* out, uint32_t seed) {
  uint32_t x[CH], y = seed * 2654435761u + threadIdx.x, z = seed ^ 0x9e3779b9u;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = seed + c * 7 + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 2) { uint32_t lo, hi;
        asm volatile("{.reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0,%1}, t;}" : "=r"(lo), "=r"(hi) : "r"(x[c]), "r"(y));
        x[c] = lo ^ hi; }
      if (OP == 3) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
      if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c];
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) {
    unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm));
    if (blockIdx.x < 2048) g_clk[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
}

// ---- modmul primitives (private copies; the product path has its own in csrc/) ----
__device__ __forceinline__ uint32_t shoup32(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
  uint32_t q = __umulhi(x, wq);
  return x * w - q * p;   // in [0, 2p)
}
__device__ __forceinline__ uint32_t mont32(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv_neg) {
  uint64_t t = (uint64_t)a * b;
  uint32_t m = (uint32_t)t * pinv_neg;
  uint64_t u = t + (uint64_t)m * p;
  return (uint32_t)(u >> 32);   // in [0, 2p)
}
__device__ __forceinline__ uint64_t gold_mul(uint64_t a, uint64_t b) {
  uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint32_t t0, t1, t2, t3;
  asm("{\n\t"
      "mul.lo.u32 %0, %4, %6;\n\t"
      "mul.hi.u32 %1, %4, %6;\n\t"
      "mad.lo.cc.u32 %1, %4, %7, %1;\n\t"
      "madc.hi.u32 %2, %4, %7, 0;\n\t"
      "mad.lo.cc.u32 %1, %5, %6, %1;\n\t"
      "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
      "madc.hi.u32 %3, %5, %7, 0;\n\t"
      "mad.lo.cc.u32 %2, %5, %7, %2;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "}" : "=r"(t0), "=r"(t1), "=r"(t2), "=r"(t3) : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
  // t = t0 + t1 2^32 + t2 2^64 + t3 2^96 ; 2^64 = 2^32 - 1, 2^96 = -1 (mod p)
  uint64_t lo = ((uint64_t)t1 << 32) | t0;
  uint64_t r = lo - t3;
  if (lo < t3) r -= 0xffffffffull;          // borrow: + p == - (2^32 - 1) mod 2^64
  uint64_t m = ((uint64_t)t2 << 32) - t2;  // t2 * (2^32 - 1)
  uint64_t s = r + m;
  if (s < m) s += 0xffffffffull;            // carry: 2^64 == 2^32 - 1
  return s;
}

template <int OP>
__global__ void __launch_bounds__(512) k_mod(uint32_t* out, uint32_t seed) {
  const uint32_t p = 998244353u;
  const uint32_t w = 3u + seed, wq = (uint32_t)(((uint64_t)w << 32) / p);
  const uint32_t pinv_neg = 998244351u;  // -p^{-1} mod 2^32 for p = 998244353
  uint32_t x[CH];
  uint64_t g[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = seed + c * 7 + threadIdx.x; g[c] = ((uint64_t)x[c] << 29) ^ x[c]; }
  const uint64_t gw = 0x123456789abcdefull + seed;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) x[c] = shoup32(x[c], w, wq, p);
      if (OP == 1) x[c] = mont32(x[c], x[(c + 1) % CH] | 1u, p, pinv_neg);
      if (OP == 2) g[c] = gold_mul(g[c], gw);
      if (OP == 3) {  // a Harvey-style Shoup butterfly pair on (x[c], x[c^1])
        if ((c & 1) == 0) {
          uint32_t X = x[c], Y = x[c + 1];
          X = min(X, X - 2 * p);
          uint32_t T = shoup32(Y, w, wq, p);
          x[c] = X + T; x[c + 1] = X - T + 2 * p;
        }
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ (uint32_t)g[c] ^ (uint32_t)(g[c] >> 32);
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x < 2048) g_clk[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <typename K>
static int run(const char* name, K kern, double ops_per_chain_iter, int nsm, uint32_t* d_out) {
  const int threads = 512, blocks = nsm * 2;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(d_out, 1u); CK(cudaDeviceSynchronize());
  float best = 1e30f; double clk_mhz = 0;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0)); kern<<<blocks, threads>>>(d_out, (uint32_t)r + 2); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) {
      best = ms;
      unsigned long long h[2048]; CK(cudaMemcpyFromSymbol(h, g_clk, sizeof(unsigned long long) * blocks));
      unsigned long long mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
      clk_mhz = (double)mx / (ms * 1e3);  // cycles per microsecond (upper bound of in-kernel time)
    }
  }
  double ops = ops_per_chain_iter * CH * (double)ITERS * threads * blocks;
  double per_s = ops / (best * 1e-3);
  double per_sm_clk = per_s / nsm / (clk_mhz * 1e6);
  printf("{\"bench\": \"%s\", \"ms\": %.4f, \"ops_per_s\": %.4e, \"per_sm_per_clk\": %.2f, \"clk_mhz_est\": %.0f}\n",
         name, best, per_s, per_sm_clk, clk_mhz);
  return 0;
}

int main() {
  int dev = 0, nsm = 0; CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"l2_bytes\": %d, \"smem_optin\": %zu}\n",
         prop.name, nsm, prop.major, prop.minor, prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  uint32_t* d_out; CK(cudaMalloc(&d_out, 64));
  run("imad_lo", k_raw<0>, 1, nsm, d_out);
  run("imad_hi", k_raw<1>, 1, nsm, d_out);
  run("imad_wide_u32(+xor)", k_raw<2>, 1, nsm, d_out);
  run("iadd3", k_raw<3>, 1, nsm, d_out);
  run("lop3", k_raw<4>, 1, nsm, d_out);
  run("shoup32_modmul", k_mod<0>, 1, nsm, d_out);
  run("mont32_modmul", k_mod<1>, 1, nsm, d_out);
  run("gold64_modmul", k_mod<2>, 1, nsm, d_out);
  run("shoup32_butterfly(per modmul)", k_mod<3>, 0.5, nsm, d_out);
  return 0;
}

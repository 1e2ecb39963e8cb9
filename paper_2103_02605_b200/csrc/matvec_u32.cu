// matvec_u32.cu — the f-circulant product executor for the 32-bit NTT primes (FieldU32).
#include "matvec_impl.cuh"

namespace fcirc {

int run_matvec_u32(const FieldU32& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                   int64_t batch, cudaStream_t st, int dev, const EmbedIO& io) {
  return run_matvec(fld, dp, a, b, c, L, batch, st, dev, io);
}

int split_log_n_u32(int L) { return msplit<FieldU32>(L); }

}  // namespace fcirc

// matvec_m31.cu — the f-circulant product executor for the paper's own ring Z/pZ[sqrt 3],
// p = 2^31 - 1 (FieldM31x2, packed 64-bit elements).
#include "matvec_impl.cuh"

namespace fcirc {

int run_matvec_m31(const FieldM31x2& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                   int64_t batch, cudaStream_t st, int dev, const EmbedIO& io) {
  return run_matvec(fld, dp, a, b, c, L, batch, st, dev, io);
}

int split_log_n_m31(int L) { return msplit<FieldM31x2>(L); }

}  // namespace fcirc

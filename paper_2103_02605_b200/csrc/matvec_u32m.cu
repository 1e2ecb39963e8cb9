// matvec_u32m.cu — the multi-prime executor (FieldU32M): bigint_mul's three 32-bit CRT products as
// one launch per pass (fcirc_kernels.cuh MultiPrime).
#include "matvec_impl.cuh"

namespace fcirc {

int run_matvec_u32m(const DevPlan& dp, const void* a, const void* b, void* c, int L, int64_t batch,
                    cudaStream_t st, int dev, const EmbedIO& io, const MultiPrime& mp) {
  FieldU32M fld;
  static_cast<FieldU32&>(fld) = mp.ps[0].fld;
  return run_matvec(fld, dp, a, b, c, L, batch, st, dev, io, &mp);
}

}  // namespace fcirc

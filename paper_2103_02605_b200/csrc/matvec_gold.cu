// matvec_gold.cu — the f-circulant product executor for Goldilocks p = 2^64 - 2^32 + 1 (FieldGold).
#include "matvec_impl.cuh"

namespace fcirc {

int run_matvec_gold(const FieldGold& fld, const DevPlan& dp, const void* a, const void* b, void* c, int L,
                    int64_t batch, cudaStream_t st, int dev, const EmbedIO& io) {
  return run_matvec(fld, dp, a, b, c, L, batch, st, dev, io);
}

int max_log_n(int kind) {
  return (kind == KIND_U32 ? FTraits<FieldU32>::MMAX : FTraits<FieldGold>::MMAX) + KMAX;   // M31: 13 as Gold
}
int split_log_n(int kind, int L) {
  return kind == KIND_GOLD ? msplit<FieldGold>(L) : kind == KIND_M31X2 ? split_log_n_m31(L) : split_log_n_u32(L);
}

}  // namespace fcirc

// Instantiation of the shared-memory-resident CG kernels (small-problem regime, kcg_res.cuh), K = 5..8,
// and the dispatchers.
#include "kcg_res.cuh"

namespace kcg {
template struct ResEntry<5>;
template struct ResEntry<6>;
template struct ResEntry<7>;
template struct ResEntry<8>;
extern template struct ResEntry<1>;
extern template struct ResEntry<2>;
extern template struct ResEntry<3>;
extern template struct ResEntry<4>;

#define KCG_RES_DISPATCH(K, CALL)                  \
  switch (K) {                                     \
    case 1: { constexpr int KK = 1; CALL; } break; \
    case 2: { constexpr int KK = 2; CALL; } break; \
    case 3: { constexpr int KK = 3; CALL; } break; \
    case 4: { constexpr int KK = 4; CALL; } break; \
    case 5: { constexpr int KK = 5; CALL; } break; \
    case 6: { constexpr int KK = 6; CALL; } break; \
    case 7: { constexpr int KK = 7; CALL; } break; \
    case 8: { constexpr int KK = 8; CALL; } break; \
    default: return cudaErrorInvalidValue;         \
  }

size_t res_smem(int K, int RS, int side, bool hits, bool prec, int n_sys) {
  return res_smem_bytes(K, RS, side, hits, prec, n_sys);
}
cudaError_t res_kernel_config(int K, bool hits, bool prec, size_t smem, int* blocks_per_sm) {
  KCG_RES_DISPATCH(K, return ResEntry<KK>::config(hits, prec, smem, blocks_per_sm));
  return cudaErrorInvalidValue;
}
cudaError_t launch_cg_resident(int K, bool prec, cudaStream_t s, const CgArgs& a, double* part, int grid, size_t smem) {
  KCG_RES_DISPATCH(K, return ResEntry<KK>::launch(prec, s, a, part, grid, smem));
  return cudaErrorInvalidValue;
}
}  // namespace kcg

// Instantiation of the textbook (HS) CG variant kernels for K = 5..8 (kcg_hs.cuh) and the dispatchers.
#include "kcg_hs.cuh"

namespace kcg {
template struct HsEntry<5>;
template struct HsEntry<6>;
template struct HsEntry<7>;
template struct HsEntry<8>;
extern template struct HsEntry<1>;
extern template struct HsEntry<2>;
extern template struct HsEntry<3>;
extern template struct HsEntry<4>;

#define KCG_HS_DISPATCH(K, CALL)                   \
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

cudaError_t hs_kernel_config(int K, bool hits, bool prec, bool d2, int n_sys, int* max_grid, size_t* smem) {
  KCG_HS_DISPATCH(K, return HsEntry<KK>::config(hits, prec, d2, n_sys, max_grid, smem));
  return cudaErrorInvalidValue;
}
cudaError_t launch_cg_hs(int K, bool prec, bool d2, cudaStream_t s, const CgArgs& a, double* q, double* part,
                         int grid, size_t smem) {
  KCG_HS_DISPATCH(K, return HsEntry<KK>::launch(prec, d2, s, a, q, part, grid, smem));
  return cudaErrorInvalidValue;
}
cudaError_t launch_hs_xfix(int K, cudaStream_t s, const SysState* st, const double* p0, const double* p1, double* x,
                           int n_sys, int side, int pitch) {
  KCG_HS_DISPATCH(K, return HsEntry<KK>::xfix(s, st, p0, p1, x, n_sys, side, pitch));
  return cudaErrorInvalidValue;
}
}  // namespace kcg

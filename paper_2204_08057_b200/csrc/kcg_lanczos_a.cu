// Instantiation of the block-Lanczos kernels for K = 1..4, and the K dispatch.
#include "kcg_lanczos.cuh"

namespace kcg {
template struct LzEntry<1>;
template struct LzEntry<2>;
template struct LzEntry<3>;
template struct LzEntry<4>;
extern template struct LzEntry<5>;  // kcg_lanczos_b.cu
extern template struct LzEntry<6>;
extern template struct LzEntry<7>;
extern template struct LzEntry<8>;

#define KCG_LZ_DISPATCH(call)          \
  switch (K) {                          \
    case 1: return LzEntry<1>::call;    \
    case 2: return LzEntry<2>::call;    \
    case 3: return LzEntry<3>::call;    \
    case 4: return LzEntry<4>::call;    \
    case 5: return LzEntry<5>::call;    \
    case 6: return LzEntry<6>::call;    \
    case 7: return LzEntry<7>::call;    \
    case 8: return LzEntry<8>::call;    \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t lz_kernel_config(int K, bool hits, bool d2, int* max_grid, size_t* smem) {
  KCG_LZ_DISPATCH(config(hits, d2, max_grid, smem))
}
cudaError_t launch_lanczos(int K, bool hits, bool d2, cudaStream_t s, const LzArgs& a, const CUtensorMap& vmap,
                           int grid, size_t smem) {
  KCG_LZ_DISPATCH(launch(hits, d2, s, a, vmap, grid, smem))
}
cudaError_t launch_lz_assemble(int K, cudaStream_t s, const LzArgs& a) { KCG_LZ_DISPATCH(assemble(s, a)) }
}  // namespace kcg

// Instantiation of the block-Lanczos kernels for K = 5..8.
#include "kcg_lanczos.cuh"

namespace kcg {
template struct LzEntry<5>;
template struct LzEntry<6>;
template struct LzEntry<7>;
template struct LzEntry<8>;
}  // namespace kcg

// Instantiation of the textbook (HS) CG variant kernels for K = 1..4 (kcg_hs.cuh) and its launchers.
#include "kcg_hs.cuh"

namespace kcg {
template struct HsEntry<1>;
template struct HsEntry<2>;
template struct HsEntry<3>;
template struct HsEntry<4>;
}  // namespace kcg

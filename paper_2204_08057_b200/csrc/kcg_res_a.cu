// Instantiation of the shared-memory-resident CG kernels (small-problem regime, kcg_res.cuh), K = 1..4.
#include "kcg_res.cuh"

namespace kcg {
template struct ResEntry<1>;
template struct ResEntry<2>;
template struct ResEntry<3>;
template struct ResEntry<4>;
}  // namespace kcg

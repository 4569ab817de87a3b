// Instantiation of the persistent CG kernels for K = 4 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<4>;
}  // namespace kcg

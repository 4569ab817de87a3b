// Instantiation of the persistent CG kernels for K = 7 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<7>;
}  // namespace kcg

// Instantiation of the persistent CG kernels for K = 2 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<2>;
}  // namespace kcg

// Instantiation of the persistent CG kernels for K = 3 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<3>;
}  // namespace kcg

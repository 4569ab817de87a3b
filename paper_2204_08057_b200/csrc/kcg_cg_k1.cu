// Instantiation of the persistent CG kernels for K = 1 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<1>;
}  // namespace kcg

// Instantiation of the persistent CG kernels for K = 6 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<6>;
}  // namespace kcg

// Instantiation of the persistent CG kernels for K = 5 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<5>;
}  // namespace kcg

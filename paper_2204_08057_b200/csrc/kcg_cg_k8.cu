// Instantiation of the persistent CG kernels for K = 8 component planes per system.
#include "kcg_cg.cuh"

namespace kcg {
template struct CgEntry<8>;
}  // namespace kcg

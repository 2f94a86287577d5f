// ln_f32.cu — LayerNorm forward/backward instantiations for float rows.
#include "ln_launch.cuh"

namespace gnsb {
GNSB_INSTANTIATE_LN(float)
}  // namespace gnsb

// ln_f64.cu — LayerNorm forward/backward instantiations for double rows.
#include "ln_launch.cuh"

namespace gnsb {
GNSB_INSTANTIATE_LN(double)
}  // namespace gnsb

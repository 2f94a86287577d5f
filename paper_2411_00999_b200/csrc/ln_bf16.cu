// ln_bf16.cu — LayerNorm forward/backward instantiations for __nv_bfloat16 rows.
#include "ln_launch.cuh"

namespace gnsb {
GNSB_INSTANTIATE_LN(__nv_bfloat16)
}  // namespace gnsb

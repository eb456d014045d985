// Persistent decode-step kernel, head_dim 64, 4 query heads per kv head.
#include "decode_step_impl.cuh"

namespace sw {
SW_DECODE_STEP_INSTANTIATE(64, 4)
}  // namespace sw

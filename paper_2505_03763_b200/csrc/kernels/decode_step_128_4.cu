// Persistent decode-step kernel, head_dim 128, 4 query heads per kv head.
#include "decode_step_impl.cuh"

namespace sw {
SW_DECODE_STEP_INSTANTIATE(128, 4)
}  // namespace sw

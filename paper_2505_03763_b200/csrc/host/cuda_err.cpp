// CUDA error -> sw::CudaError (mapped to SW_ECUDA at the C-ABI).
#include <cuda_runtime.h>

#include <string>

#include "capi_util.hpp"

namespace sw {
[[noreturn]] void throw_cuda(const char* what, cudaError_t e, const char* file, int line) {
    throw CudaError(std::string(what) + " failed: " + cudaGetErrorString(e) + " at " + file + ":" + std::to_string(line));
}
}  // namespace sw

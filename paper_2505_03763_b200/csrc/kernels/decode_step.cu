// Dispatch of the persistent decode-step kernel (decode_step_impl.cuh) over
// its instantiated (head_dim, group) configurations.
#include "common.cuh"
#include "decode_step.cuh"

namespace sw {

void decode_step_launch_64_4(const StepArgs& a, int bn, int ctas, cudaStream_t st);
void decode_step_launch_64_2(const StepArgs& a, int bn, int ctas, cudaStream_t st);
void decode_step_launch_128_4(const StepArgs& a, int bn, int ctas, cudaStream_t st);
int decode_step_stages_64_4(int bn);
int decode_step_stages_64_2(int bn);
int decode_step_stages_128_4(int bn);

bool decode_step_supported(int bn, int hd, int group) {
    const bool shape = (hd == 64 && (group == 4 || group == 2)) || (hd == 128 && group == 4);
    return shape && (bn == 32 || bn == 64 || bn == 128);
}

int decode_step_stages(int bn, int hd, int group) {
    if (!decode_step_supported(bn, hd, group)) return 0;
    if (hd == 64) return group == 4 ? decode_step_stages_64_4(bn) : decode_step_stages_64_2(bn);
    return decode_step_stages_128_4(bn);
}

void decode_step_launch(const StepArgs& a, int bn, int hd, int group, int ctas, cudaStream_t st) {
    if (!decode_step_supported(bn, hd, group))
        throw_cuda("decode_step: unsupported (row tile, head_dim, group)", cudaErrorInvalidValue, __FILE__, __LINE__);
    if (hd == 64 && group == 4) decode_step_launch_64_4(a, bn, ctas, st);
    else if (hd == 64) decode_step_launch_64_2(a, bn, ctas, st);
    else decode_step_launch_128_4(a, bn, ctas, st);
}

}  // namespace sw

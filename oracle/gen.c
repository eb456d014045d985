/* ORACLE / TEST INFRASTRUCTURE ONLY -- C restatement of the synthetic weight
 * generator in oracle/model.py (tensor_values), used to make the CPU baseline
 * start quickly at Llama shapes.  Same arithmetic: SplitMix64 draw i of
 * seed ^ (k * 0x9E3779B97F4A7C15) (splitsim/prng.hpp:14-31), 53-bit unit,
 * (2u-1)*sqrt(3/fan_in) in double -> float (RNE) -> bf16 (RNE), returned as
 * float32 values.  tests/test_oracle.py checks it against the numpy path. */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline float bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    memcpy(&f, &u, 4);
    return f;
}

void oracle_gen_tensor(uint64_t seed, int k, int64_t n, int fan_in, float* out) {
    const uint64_t tseed = seed ^ ((uint64_t)k * 0x9E3779B97F4A7C15ULL);
    const double scale = sqrt(3.0 / (double)fan_in);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t z = mix(tseed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ULL);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[i] = bf16_rne((float)((2.0 * u - 1.0) * scale));
    }
}

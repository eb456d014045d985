// Foundation layer of the split-phase engine: the error taxonomy and the
// portable SplitMix64 stream every synthetic input is drawn from.
//
// Error taxonomy follows splitsim/errors.hpp:9-30 (ConfigError/ParseError ->
// exit 2, IoError -> 3, ContractViolation -> 4, tools/splitsim.cpp:124-139) so
// callers that catch the reference's exceptions keep working.
// SplitMix64 follows splitsim/prng.hpp:10-35 bit for bit; `splitmix_at` is the
// random-access form of the same stream (the i-th draw only depends on
// seed + (i+1)*gamma), which is what lets the GPU initialise billions of
// weights in parallel and still match the CPU oracle exactly.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sw {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ContractViolation : std::logic_error {
    using std::logic_error::logic_error;
};

inline constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

// The SplitMix64 finaliser (Steele/Lea/Flood 2014).
constexpr std::uint64_t splitmix_mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// i-th output (0-based) of SplitMix64(seed) without walking the stream.
constexpr std::uint64_t splitmix_at(std::uint64_t seed, std::uint64_t i) {
    return splitmix_mix(seed + (i + 1) * kGolden);
}

class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
    std::uint64_t next_u64() {
        s_ += kGolden;
        return splitmix_mix(s_);
    }
    // Inclusive [lo, hi] by modulo (prng.hpp:23-26).
    std::int64_t next_range(std::int64_t lo, std::int64_t hi) {
        const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1ULL;
        return lo + static_cast<std::int64_t>(next_u64() % span);
    }
    // 53-bit uniform in [0,1) (prng.hpp:29-31).
    double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

private:
    std::uint64_t s_;
};

}  // namespace sw

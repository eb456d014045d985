// CUDA error -> sw::CudaError (mapped to SW_ECUDA at the C-ABI).
#include <cuda_runtime.h>

#include <string>

#include "capi_util.hpp"

#include <atomic>
#include <cstdlib>

namespace sw {
std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
std::atomic<unsigned long long> g_h2d{0}, g_d2h{0};
bool& pdl_mode() {
    thread_local bool on = false;
    return on;
}
bool pdl_allowed() {  // programmatic dependent launch in the decode step; SW_PDL=0 disables (A/B)
    static const bool ok = [] {
        const char* v = std::getenv("SW_PDL");
        return !(v && v[0] == '0');
    }();
    return ok;
}
void count_transfer(unsigned long long h2d, unsigned long long d2h) {
    g_h2d.fetch_add(h2d, std::memory_order_relaxed);
    g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}
[[noreturn]] void throw_cuda(const char* what, cudaError_t e, const char* file, int line) {
    throw CudaError(std::string(what) + " failed: " + cudaGetErrorString(e) + " at " + file + ":" + std::to_string(line));
}
}  // namespace sw

extern "C" unsigned long long sw_launch_count(void) { return sw::g_launches.load(); }
extern "C" void sw_transfer_bytes(unsigned long long* h2d, unsigned long long* d2h) {
    if (h2d) *h2d = sw::g_h2d.load();
    if (d2h) *d2h = sw::g_d2h.load();
}

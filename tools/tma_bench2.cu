// Follow-up microbenchmark: is the ~1 box / 616 cycles per SM cap on the
// issuing thread or the copy unit?  P producer warps (one lane each, own
// ring of S stages); 1D bulk copies of C bytes.  All 148 SMs or 1 SM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* base, int chunk, int stages, int iters, int64_t region, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int P = blockDim.x / 32, w = threadIdx.x / 32;
    uint64_t* full = (uint64_t*)(sm + 200 * 1024) + w * 16;
    uint8_t* ring = sm + (size_t)w * stages * chunk;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    const int64_t off0 = (int64_t)blockIdx.x * region + (int64_t)w * (region / P);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters + stages; ++it) {
        if (it >= stages) {
            const int s = (it - stages) % stages;
            const uint32_t ph = ((it - stages) / stages) & 1;
            asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(sa(&full[s])), "r"(ph));
        }
        if (it < iters) {
            const int s = it % stages;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(chunk));
            const int64_t o = off0 + ((int64_t)it * chunk) % (region / P);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(ring + s * chunk)), "l"(base + o), "r"(chunk), "r"(sa(&full[s])) : "memory");
        }
    }
    if (w == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    const int64_t total = (int64_t)2 << 30;
    uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
    unsigned long long* cyc; cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    const int64_t region = (total / 148) / 1024 * 1024;
    for (int P : {1, 2, 4})
        for (int chunk : {8192, 16384, 32768, 65536})
            for (int stages : {2, 4})
                for (int grid : {1, 148}) {
                    if ((int64_t)P * stages * chunk > 200 * 1024) continue;
                    const int iters = (int)std::min<int64_t>(4000, (region / P) / chunk);
                    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                    bulk_kernel<<<grid, 32 * P, 210 * 1024>>>(buf, chunk, stages, 20, region, cyc);
                    cudaEventRecord(e0);
                    bulk_kernel<<<grid, 32 * P, 210 * 1024>>>(buf, chunk, stages, iters, region, cyc);
                    cudaEventRecord(e1); cudaEventSynchronize(e1);
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    const double bytes = (double)iters * chunk * P;
                    std::vector<unsigned long long> c(grid); cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                    double avg = 0; for (auto x : c) avg += x; avg /= grid;
                    printf("P=%d chunk=%6d stages=%d grid=%3d : %6.1f B/cycle/SM %7.1f GB/s total\n", P, chunk, stages, grid,
                           bytes / avg, bytes * grid / (ms * 1e-3) / 1e9);
                }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

// Microbenchmark: how many SMs does it take to saturate HBM?
// Each CTA streams a private region of a 4 GB buffer global->shared with 1D
// bulk copies (P producer lanes, S stages of C bytes each in flight), and the
// grid is swept from 8 to 148 CTAs (one per SM).  This is the number that
// decides whether a decode partition of k SMs can run at full HBM speed while
// prefill holds the rest.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_sm_scaling.cu -o /tmp/hbm_sm
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const uint8_t* base, int chunk, int stages, int iters, int64_t region) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int P = blockDim.x / 32, w = threadIdx.x / 32;
    uint64_t* full = (uint64_t*)(sm + 208 * 1024) + w * 16;
    uint8_t* ring = sm + (size_t)w * stages * chunk;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    const int64_t off0 = (int64_t)blockIdx.x * region + (int64_t)w * (region / P);
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
}

// plain vector loads: T threads per CTA, U independent 16-byte loads in flight per thread
template <int U>
__global__ void ldg_kernel(const int4* base, int64_t n_per_cta, int4* sink) {
    const int4* p = base + (int64_t)blockIdx.x * n_per_cta;
    int4 acc = make_int4(0, 0, 0, 0);
    for (int64_t i = threadIdx.x; i + (U - 1) * blockDim.x < n_per_cta; i += (int64_t)U * blockDim.x) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    }
    if (acc.x == 0x12345678) sink[threadIdx.x] = acc;
}

int main() {
    const int64_t total = (int64_t)4 << 30;
    uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
    int4* sink; cudaMalloc(&sink, 4096 * 16);
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 212 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grids[] = {8, 16, 24, 32, 40, 48, 64, 80, 96, 112, 128, 148};
    printf("# bulk copies (cp.async.bulk, 1 lane per producer warp)\n");
    struct Cfg { int P, chunk, stages; };
    const Cfg cfgs[] = {{1, 32768, 6}, {2, 16384, 6}, {4, 16384, 3}, {4, 8192, 6}, {8, 8192, 3}};
    for (const Cfg& c : cfgs) {
        for (int grid : grids) {
            const int64_t region = (total / grid) / 65536 * 65536;
            const int iters = (int)std::min<int64_t>(20000, (region / c.P) / c.chunk);
            bulk_kernel<<<grid, 32 * c.P, 212 * 1024>>>(buf, c.chunk, c.stages, 16, region);
            cudaEventRecord(e0);
            bulk_kernel<<<grid, 32 * c.P, 212 * 1024>>>(buf, c.chunk, c.stages, iters, region);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)iters * c.chunk * c.P * grid;
            printf("bulk P=%d chunk=%6d stages=%d inflight=%3d KB grid=%3d : %7.1f GB/s  (%5.1f GB/s/SM)\n", c.P, c.chunk,
                   c.stages, c.P * c.chunk * c.stages / 1024, grid, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / grid);
        }
    }
    printf("# LDG.128 streaming (__ldcs), 1024 threads x 8 loads in flight, 1 CTA per SM\n");
    for (int grid : grids) {
        const int ctas = grid;
        const int64_t n_per = (total / 16 / ctas) / 8192 * 8192;
        ldg_kernel<8><<<ctas, 1024>>>((const int4*)buf, n_per, sink);
        cudaEventRecord(e0);
        ldg_kernel<8><<<ctas, 1024>>>((const int4*)buf, n_per, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)n_per * 16 * ctas;
        printf("ldg U=8 grid=%3d SMs : %7.1f GB/s  (%5.1f GB/s/SM)\n", grid, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / grid);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

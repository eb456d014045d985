// Microbenchmark: global->shared streaming rate per SM on B200 for
//   (a) 2D tiled TMA (cp.async.bulk.tensor, SWIZZLE_128B, box 64 x R bf16)
//   (b) 1D bulk copy (cp.async.bulk, contiguous chunk)
// with S stages in flight, one producer thread, consumer releases at once.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_bench.cu -o /tmp/tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool BULK>
__global__ void stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* base, int rows_box, int stages,
                              int iters, int64_t region_rows, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + 200 * 1024);
    const int box_bytes = rows_box * 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int64_t row0 = (int64_t)blockIdx.x * region_rows;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters + stages; ++it) {
        if (it >= stages) {  // consume it - stages
            const int s = (it - stages) % stages;
            const uint32_t ph = ((it - stages) / stages) & 1;
            asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(sa(&full[s])), "r"(ph));
        }
        if (it < iters) {
            const int s = it % stages;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(box_bytes));
            const int64_t r = row0 + ((int64_t)it * rows_box) % region_rows;  // unique rows: DRAM, not L2
            if (BULK) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + s * box_bytes)), "l"(base + r * 128), "r"(box_bytes), "r"(sa(&full[s])) : "memory");
            } else {
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(sa(sm + s * box_bytes)), "l"(&tm), "r"(0), "r"((int)r), "r"(sa(&full[s])) : "memory");
            }
        }
    }
    cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int64_t total_rows = (int64_t)1 << 24;  // 16M rows x 128 B = 2 GB
    uint8_t* buf;
    CK(cudaMalloc(&buf, total_rows * 128));
    CK(cudaMemset(buf, 1, total_rows * 128));
    void* fp; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    unsigned long long* cyc;
    CK(cudaMalloc(&cyc, 148 * 8));
    for (auto fn : {stream_kernel<false>, stream_kernel<true>})
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    for (int bulk = 0; bulk < 2; ++bulk)
        for (int rows_box : {64, 128, 256})
            for (int stages : {2, 4, 8})
                for (int grid : {1, 16, 148}) {
                    if (stages * rows_box * 128 > 200 * 1024) continue;
                    CUtensorMap tm;
                    cuuint64_t dims[2] = {64, (cuuint64_t)total_rows};
                    cuuint64_t strides[1] = {128};
                    cuuint32_t box[2] = {64, (cuuint32_t)rows_box};
                    cuuint32_t es[2] = {1, 1};
                    ((EncFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    const int iters = (int)std::min<int64_t>(2000, (total_rows / 148) / rows_box);
                    const int64_t region = total_rows / 148;
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0); cudaEventCreate(&e1);
                    auto fn = bulk ? stream_kernel<true> : stream_kernel<false>;
                    fn<<<grid, 32, 210 * 1024>>>(tm, buf, rows_box, stages, 50, region, cyc);
                    cudaEventRecord(e0);
                    fn<<<grid, 32, 210 * 1024>>>(tm, buf, rows_box, stages, iters, region, cyc);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    std::vector<unsigned long long> c(grid);
                    cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                    double avg = 0; for (auto x : c) avg += x; avg /= grid;
                    const double bytes = (double)iters * rows_box * 128;
                    printf("%s box_rows=%3d stages=%d grid=%3d : %6.1f B/cycle/SM  %7.1f GB/s total  (%.1f us)\n",
                           bulk ? "bulk1d" : "tma2d ", rows_box, stages, grid, bytes / avg, bytes * grid / (ms * 1e-3) / 1e9, ms * 1e3);
                }
    return 0;
}

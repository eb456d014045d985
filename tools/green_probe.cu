// Probe: green-context SM partitions driven through the CUDA runtime API, the
// way the split executor uses them.  Checks (1) kernels launched with the
// runtime into a green-context stream stay on that partition's SMs, (2) events
// created in the primary context can be recorded on green streams and timed
// against each other, (3) a graph captured on a green stream replays there,
// (4) memory from the primary context is usable.
//   nvcc -std=c++17 -arch=sm_100a -o /tmp/green_probe tools/green_probe.cu -lcuda && /tmp/green_probe 48
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        CUresult r_ = (x);                                                             \
        if (r_ != CUDA_SUCCESS) {                                                      \
            const char* s_ = nullptr;                                                  \
            cuGetErrorString(r_, &s_);                                                 \
            std::printf("FAIL %s: %s\n", #x, s_ ? s_ : "?");                           \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)
#define CR(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_));                  \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

__global__ void smid_kernel(int* out, int spin) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(s);
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
}

static std::set<int> sms_of(const std::vector<int>& v) { return std::set<int>(v.begin(), v.end()); }

int main(int argc, char** argv) {
    const int want = argc > 1 ? std::atoi(argv[1]) : 48;
    CR(cudaFree(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    CUdevResource grp, rest;
    unsigned n = 1;
    CK(cuDevSmResourceSplitByCount(&grp, &n, &all, &rest, 0, want));
    std::printf("device SMs %u -> group %u SMs, remaining %u SMs\n", all.sm.smCount, grp.sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dg, dr;
    CK(cuDevResourceGenerateDesc(&dg, &grp, 1));
    CK(cuDevResourceGenerateDesc(&dr, &rest, 1));
    CUgreenCtx gg, gr;
    CK(cuGreenCtxCreate(&gg, dg, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sg, sr;
    CK(cuGreenCtxStreamCreate(&sg, gg, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&sr, gr, CU_STREAM_NON_BLOCKING, 0));

    const int blocks = 1024;
    int *dg_out, *dr_out;
    CR(cudaMalloc(&dg_out, blocks * 4));
    CR(cudaMalloc(&dr_out, blocks * 4));
    cudaEvent_t e0, e1, e2;
    CR(cudaEventCreate(&e0));
    CR(cudaEventCreate(&e1));
    CR(cudaEventCreate(&e2));
    CR(cudaEventRecord(e0, (cudaStream_t)sr));
    smid_kernel<<<blocks, 64, 0, (cudaStream_t)sg>>>(dg_out, 200000);
    CR(cudaGetLastError());
    smid_kernel<<<blocks, 64, 0, (cudaStream_t)sr>>>(dr_out, 200000);
    CR(cudaGetLastError());
    CR(cudaEventRecord(e1, (cudaStream_t)sg));
    CR(cudaEventRecord(e2, (cudaStream_t)sr));
    CR(cudaDeviceSynchronize());
    std::vector<int> hg(blocks), hr(blocks);
    CR(cudaMemcpy(hg.data(), dg_out, blocks * 4, cudaMemcpyDeviceToHost));
    CR(cudaMemcpy(hr.data(), dr_out, blocks * 4, cudaMemcpyDeviceToHost));
    auto a = sms_of(hg), b = sms_of(hr);
    int overlap = 0;
    for (int s : a) overlap += b.count(s);
    std::printf("group kernel used %zu SMs, rest kernel used %zu SMs, overlap %d\n", a.size(), b.size(), overlap);
    float ms1 = 0, ms2 = 0;
    CR(cudaEventElapsedTime(&ms1, e0, e1));
    CR(cudaEventElapsedTime(&ms2, e0, e2));
    std::printf("cross-stream event timing ok: %.3f ms / %.3f ms\n", ms1, ms2);

    // graph captured on the group stream, replayed there
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    CR(cudaStreamBeginCapture((cudaStream_t)sg, cudaStreamCaptureModeThreadLocal));
    smid_kernel<<<blocks, 64, 0, (cudaStream_t)sg>>>(dg_out, 1000);
    CR(cudaStreamEndCapture((cudaStream_t)sg, &graph));
    CR(cudaGraphInstantiate(&exec, graph, 0));
    CR(cudaMemset(dg_out, 0xff, blocks * 4));
    CR(cudaGraphLaunch(exec, (cudaStream_t)sg));
    CR(cudaStreamSynchronize((cudaStream_t)sg));
    CR(cudaMemcpy(hg.data(), dg_out, blocks * 4, cudaMemcpyDeviceToHost));
    auto c = sms_of(hg);
    int outside = 0;
    for (int s : c) outside += a.count(s) ? 0 : 1;
    std::printf("graph replay on group stream used %zu SMs, %d outside the group\n", c.size(), outside);
    // graph captured on a primary-context stream, launched into the group stream
    cudaStream_t ps;
    CR(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
    CR(cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal));
    smid_kernel<<<blocks, 64, 0, ps>>>(dg_out, 1000);
    CR(cudaStreamEndCapture(ps, &graph));
    CR(cudaGraphInstantiate(&exec, graph, 0));
    CR(cudaGraphLaunch(exec, (cudaStream_t)sg));
    CR(cudaStreamSynchronize((cudaStream_t)sg));
    CR(cudaMemcpy(hg.data(), dg_out, blocks * 4, cudaMemcpyDeviceToHost));
    auto d = sms_of(hg);
    outside = 0;
    for (int s : d) outside += a.count(s) ? 0 : 1;
    std::printf("primary-captured graph launched on group stream used %zu SMs, %d outside the group\n", d.size(), outside);
    std::printf("OK\n");
    return 0;
}

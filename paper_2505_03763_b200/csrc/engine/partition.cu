// Green-context SM partitions (see partition.hpp).  Measured on B200
// (tools/green_probe.cu): runtime launches into a green stream stay on its
// SMs, primary-context events time across green streams, and a CUDA graph is
// confined to a partition only when it is captured on that partition's stream.
#include <cuda.h>

#include <map>
#include <mutex>
#include <string>

#include "../host/capi_util.hpp"
#include "../kernels/common.cuh"
#include "partition.hpp"

namespace sw {

namespace {

struct Driver {
    CUresult (*deviceGet)(CUdevice*, int) = nullptr;
    CUresult (*getDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
    CUresult (*splitByCount)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned) = nullptr;
    CUresult (*generateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
    CUresult (*greenCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
    CUresult (*greenStream)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
    CUresult (*greenDestroy)(CUgreenCtx) = nullptr;
};

template <class F>
void resolve(F& fn, const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    SW_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw ConfigError(std::string("green contexts: driver lacks ") + name);
    fn = reinterpret_cast<F>(p);
}

const Driver& driver() {
    static const Driver d = [] {
        Driver x;
        resolve(x.deviceGet, "cuDeviceGet");
        resolve(x.getDevResource, "cuDeviceGetDevResource");
        resolve(x.splitByCount, "cuDevSmResourceSplitByCount");
        resolve(x.generateDesc, "cuDevResourceGenerateDesc");
        resolve(x.greenCreate, "cuGreenCtxCreate");
        resolve(x.greenStream, "cuGreenCtxStreamCreate");
        resolve(x.greenDestroy, "cuGreenCtxDestroy");
        return x;
    }();
    return d;
}

void ck(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw CudaError(std::string("green contexts: ") + what + " failed (CUresult " + std::to_string(r) + ")");
}

std::mutex g_mu;
std::map<std::tuple<int, int, int>, SmPartition> g_parts;  // (device, decode_sms, lanes)
std::map<cudaStream_t, int> g_stream_sms;

}  // namespace

const SmPartition& sm_partition(int device, int decode_sms, int lanes) {
    std::lock_guard<std::mutex> lk(g_mu);
    const auto key = std::make_tuple(device, decode_sms, lanes);
    auto it = g_parts.find(key);
    if (it != g_parts.end()) return it->second;
    const Driver& D = driver();
    SW_CUDA(cudaSetDevice(device));
    SW_CUDA(cudaFree(nullptr));  // primary context up
    CUdevice dev;
    ck(D.deviceGet(&dev, device), "cuDeviceGet");
    CUdevResource all{};
    ck(D.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
    if (decode_sms < 8 || decode_sms > static_cast<int>(all.sm.smCount) - 8)
        throw ConfigError("engine.decode_sms must leave >= 8 SMs to each phase (device has " +
                          std::to_string(all.sm.smCount) + ")");
    CUdevResource grp{}, rest{};
    unsigned n = 1;
    ck(D.splitByCount(&grp, &n, &all, &rest, 0, static_cast<unsigned>(decode_sms)), "cuDevSmResourceSplitByCount");
    if (n != 1) throw ConfigError("engine.decode_sms: the SM split produced no group");
    CUdevResourceDesc dd{}, dp{};
    ck(D.generateDesc(&dd, &grp, 1), "cuDevResourceGenerateDesc(decode)");
    ck(D.generateDesc(&dp, &rest, 1), "cuDevResourceGenerateDesc(prefill)");
    CUgreenCtx gd{}, gp{};
    ck(D.greenCreate(&gd, dd, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate(decode)");
    ck(D.greenCreate(&gp, dp, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate(prefill)");
    int lo = 0, hi = 0;
    SW_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SmPartition P;
    P.requested_decode_sms = decode_sms;
    P.decode_sms = static_cast<int>(grp.sm.smCount);
    P.prefill_sms = static_cast<int>(rest.sm.smCount);
    P.green_decode = gd;
    P.green_prefill = gp;
    CUstream s{};
    ck(D.greenStream(&s, gp, CU_STREAM_NON_BLOCKING, lo), "cuGreenCtxStreamCreate(prefill)");
    P.prefill = reinterpret_cast<cudaStream_t>(s);
    g_stream_sms[P.prefill] = P.prefill_sms;
    for (int i = 0; i < lanes; ++i) {
        ck(D.greenStream(&s, gd, CU_STREAM_NON_BLOCKING, hi), "cuGreenCtxStreamCreate(decode)");
        P.decode.push_back(reinterpret_cast<cudaStream_t>(s));
        g_stream_sms[P.decode.back()] = P.decode_sms;
    }
    return g_parts.emplace(key, P).first->second;
}

void sm_partitions_release() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& [k, P] : g_parts) {
        cudaStreamSynchronize(P.prefill);
        cudaStreamDestroy(P.prefill);
        for (cudaStream_t s : P.decode) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
        if (P.green_decode) driver().greenDestroy(static_cast<CUgreenCtx>(P.green_decode));
        if (P.green_prefill) driver().greenDestroy(static_cast<CUgreenCtx>(P.green_prefill));
    }
    g_parts.clear();
    g_stream_sms.clear();
}

const void* stream_partition_tag(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const auto& [k, P] : g_parts) {
        if (P.prefill == st) return P.green_prefill;
        for (cudaStream_t s : P.decode)
            if (s == st) return P.green_decode;
    }
    return nullptr;
}

int stream_sm_count(cudaStream_t st) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_stream_sms.find(st);
        if (it != g_stream_sms.end()) return it->second;
    }
    static const int n = [] {
        int dev = 0, v = 0;
        SW_CUDA(cudaGetDevice(&dev));
        SW_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

}  // namespace sw

// C-ABI (include/splitwise.h): the streams of a cached partition, for tools
// and tests that enqueue prefill/decode on one SM group directly.
extern "C" int sw_sm_partition(int device, int decode_sms, void** decode_stream, void** prefill_stream,
                               int* decode_sms_out, int* prefill_sms_out) {
    return sw::guarded([&] {
        const sw::SmPartition& P = sw::sm_partition(device, decode_sms, 1);
        if (decode_stream) *decode_stream = P.decode.front();
        if (prefill_stream) *prefill_stream = P.prefill;
        if (decode_sms_out) *decode_sms_out = P.decode_sms;
        if (prefill_sms_out) *prefill_sms_out = P.prefill_sms;
    });
}

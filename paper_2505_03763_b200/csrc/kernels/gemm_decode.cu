// Decode projection GEMM for sm_100a: swap-AB tcgen05 with split-K over a
// thread-block cluster and a column-distributed, deterministic reduction.
//
//   Y[t, f] = sum_k X[t, k] W[f, k]   W: weights bf16 [F, K] (UMMA M = 128 rows)
//                                     X: decode rows bf16 [BN, K] (UMMA N = BN)
//
// A decode step at b <= 256 rows is a weight stream, and its per-layer
// projections are narrow (Llama-1B: Wo/Wd have d/128 = 16 weight tiles), so one
// CTA per 128-row tile leaves most SMs idle.  Here tile f is split over the S
// CTAs of one cluster (S from the weight shape only, never the batch, so the
// summation order is batch invariant):
//   * CTA rank r streams K-blocks [r*nk/S, (r+1)*nk/S) into its own TMEM
//     accumulator (warp 0/1 TMA producers, warp 2 MMA issuer);
//   * the partial tile goes token-major to an L2-resident scratch
//     [tile][rank][token][128] (a warp stores 128 contiguous bytes per token),
//     then one cluster barrier;
//   * rank r owns tokens [r*n/S, (r+1)*n/S): one warp per token adds the S
//     partials in rank order (float4 per lane) and runs the fused epilogue
//     (emit_tok) on them.  Every output element is produced by exactly one
//     CTA; the reduction work is spread over all S CTAs.
// With S = 1 the accumulator is transposed through shared memory into the
// same warp-per-token epilogue.
// Shared memory is kept near 110 KB so a kernel and its successor fit on one
// SM together: under programmatic dependent launch the successor's weight
// ring fills (weights are constant) while this kernel drains.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_sm100.cuh"
#include "gemm_decode_epi.cuh"

namespace sw {

namespace {

using namespace dec_epi;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 224;  // 7 warps: 2 producers, MMA, 4 epilogue
constexpr int kEpiWarp0 = 3;
constexpr int kMaxSplit = 8;   // portable cluster size

// diagnostic (SW_DEC_TRACE=1): per-CTA globaltimer stamps of the last traced launch
// [start, last MMA issued, partials stored / cluster joined, exit] (tools/dsk_trace.py --cluster)
__device__ unsigned long long g_dec_trace[512][4];
__device__ __forceinline__ unsigned long long dec_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int BN>
struct DecCfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    // <= ~112 KB for every BN: two CTAs per SM (BN = 256: 2 stages of 48 KB each, so the 8B gate/up grid of
    // 224 CTAs and the split-K QKV / Wo / Wd grids run in one wave instead of two)
    static constexpr int kBudget = 112 * 1024;
    static constexpr int kFixed = 1024 + 256 * 16 + 256;
    static constexpr int kStagesRaw = (kBudget - kFixed) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static_assert(kStages >= 2, "stage ring too shallow");
    static constexpr int kRing = kStages * kStageBytes;
    static_assert(kRing >= 2 * 32 * (BM + 4) * 4, "epilogue transpose buffers alias the drained ring");
    static constexpr int kSmem = kFixed + kRing;
    static constexpr int kTmemCols = BN < 32 ? 32 : BN;
};

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_decode_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    using C = DecCfg<BN>;
    constexpr int NS = C::kStages;
    constexpr int kTs = BM + 4;  // token-major transpose row stride (floats): conflict-free, 16 B aligned
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + NS * C::kABytes;
    float* xt = reinterpret_cast<float*>(smem);  // [2][32][kTs] transpose buffers, alias the drained ring
    float* tok_inv = reinterpret_cast<float*>(smem + C::kRing);
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tok_inv) + 256 * 16);
    uint64_t* empty = full + NS;
    uint64_t* acc_ready = empty + NS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    griddep_launch_dependents();  // the successor may become resident and prefetch its weights
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = static_cast<int>(gridDim.x);  // cluster spans x
    const int rank = static_cast<int>(blockIdx.x);
    const int tile = static_cast<int>(blockIdx.y);
    const int trace_id = args.trace ? tile * S + rank : -1;
    if (trace_id >= 0 && trace_id < 512 && threadIdx.x == 0) g_dec_trace[trace_id][0] = dec_gtimer();
    const int m0 = tile * BM;
    const int nk_total = args.K / BK;
    const int kb0 = rank * nk_total / S;
    const int nk = (rank + 1) * nk_total / S - kb0;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_ready, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 2) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 2) {
        // -------------------------------------------------------- producers
        // K-blocks alternate between the two producer threads
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_x = l2_policy_evict_last();
            // weights are constant: fill the ring before the predecessor is done
            for (int i = warp; i < nk && i < NS; i += 2) {
                mbar_expect_tx(&full[i], C::kStageBytes);
                tma_load_2d(sA + i * C::kABytes, &tmA, &full[i], (kb0 + i) * BK, m0, pol_w);
            }
            griddep_wait();  // activations come from the predecessor
            for (int i = warp; i < nk; i += 2) {
                const int s = i % NS;
                if (i >= NS) {
                    mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
                    mbar_expect_tx(&full[s], C::kStageBytes);
                    tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], (kb0 + i) * BK, m0, pol_w);
                }
                tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], (kb0 + i) * BK, 0, pol_x);
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // -------------------------------------------------------- MMA issuer
        if (lane == 0) {
            // UMMA N trimmed to the live rows (multiple of 16): a bucket of BN rows computes only the
            // columns in use; each output column's K order is unchanged (results bit-identical)
            // (the count is loaded now and used after the first stage lands, so its latency hides there)
            griddep_wait();  // the live row count comes from the predecessor
            const int live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
            uint32_t idesc = 0;
            for (int i = 0; i < nk; ++i) {
                const int s = i % NS;
                mbar_wait(&full[s], (i / NS) & 1);
                if (i == 0) idesc = umma_idesc_bf16(BM, min(BN, max(16, (live + 15) & ~15)));
                tc_fence_after();
                const uint32_t a0 = smem_addr(sA + s * C::kABytes);
                const uint32_t b0 = smem_addr(sB + s * C::kBBytes);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                              (i | k) != 0 ? 1u : 0u);
                umma_commit(&empty[s]);
            }
            umma_commit(acc_ready);
            if (trace_id >= 0 && trace_id < 512) g_dec_trace[trace_id][1] = dec_gtimer();
        }
        __syncwarp();
    }

    const int quarter = warp & 3;         // TMEM lanes [32*quarter, +32)
    const int row = quarter * 32 + lane;  // weight row in the tile
    const int ew = warp - kEpiWarp0;      // epilogue warp 0..3
    const int e = threadIdx.x - kEpiWarp0 * 32;
    int n_live = 0;
    // split-K partials, token-major: [tile][rank][BN tokens][128 features]
    float* ws_tile = args.ws + static_cast<size_t>(tile) * S * BN * BM;
    const TokCtx tc{&args, tok_inv, tok_pos, tok_kv, m0};
    if (warp >= kEpiWarp0) {
        // -------------------------------------------------------- epilogue
        griddep_wait();
        n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        const DecodeFusion& fx = args.fx;
        // per-token inputs, gathered while the MMAs run (loads in flight together)
        for (int t = e; t < BN && t < n_live; t += 128) {
            if (fx.ss_parts) {
                float ss = 0.f;
                for (int q0 = 0; q0 < fx.ss_nparts; q0 += 16) {
                    float p[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        p[q] = q0 + q < fx.ss_nparts ? __ldcg(fx.ss_parts + (q0 + q) * kSsStride + t) : 0.f;
#pragma unroll
                    for (int q = 0; q < 16; ++q) ss += p[q];  // fixed order: deterministic
                }
                tok_inv[t] = rsqrtf(ss / static_cast<float>(fx.norm_dim) + fx.norm_eps);
            }
            if constexpr (MODE == EPI_QKV_ROPE) {
                const int pos = fx.pos[t];
                const int page = fx.page_table[static_cast<int64_t>(fx.slot[t]) * fx.max_pages + pos / fx.page_tokens];
                tok_pos[t] = pos;
                tok_kv[t] = static_cast<long long>(page) * fx.page_stride +
                            static_cast<long long>(pos % fx.page_tokens) * fx.hd;
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        mbar_wait(acc_ready, 0);
        tc_fence_after();
        const uint32_t tb = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t r[32];
        if (S == 1) {
            // TMEM (thread = feature) -> smem token-major -> one warp per token
            for (int c = 0, buf = 0; c < BN && c < n_live; c += 32, buf ^= 1) {
                tmem_ld32(tb + c, r);
                tmem_ld_wait();
                float* T = xt + buf * 32 * kTs;
#pragma unroll
                for (int j = 0; j < 32; ++j) T[j * kTs + row] = __uint_as_float(r[j]);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const int cnt = min(32, n_live - c);
                for (int j = ew; j < cnt; j += 4)
                    emit_tok<MODE>(tc, c + j, lane, *reinterpret_cast<const float4*>(T + j * kTs + 4 * lane),
                                   pre_tok<MODE>(tc, c + j, lane));
            }
        } else {
            // park this rank's partial token-major (a warp stores 128 contiguous bytes per token)
            float* part = ws_tile + static_cast<size_t>(rank) * BN * BM;
            for (int c = 0; c < BN && c < n_live; c += 32) {
                tmem_ld32(tb + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (c + j < n_live) __stcg(part + static_cast<size_t>(c + j) * BM + row, __uint_as_float(r[j]));
            }
        }
        tc_fence_before();
    }
    if (S > 1) {
        cluster_sync_all();  // every rank's partial is in L2
        if (trace_id >= 0 && trace_id < 512 && threadIdx.x == 0) g_dec_trace[trace_id][2] = dec_gtimer();
        // rank r owns tokens [r*n/S, (r+1)*n/S): add the S partials in rank order
        // (deterministic).  All warps of the CTA take part (the producer and MMA
        // warps are idle by now; the cluster barrier published the epilogue
        // warps' shared token tables to them), and the next token's loads
        // are issued before this token's stores, so a warp has two tokens of
        // L2 reads in flight instead of one dependent round trip per token.
        if (warp < kEpiWarp0) {
            griddep_wait();  // no-op by now; orders the live-token read after the predecessor
            n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        }
        const int t0 = rank * n_live / S, t1 = (rank + 1) * n_live / S;
        constexpr int kWarps = kThreads / 32;
        float4 in[kMaxSplit];
        TokPre pre{};
        auto load = [&](int t) {
#pragma unroll
            for (int k = 0; k < kMaxSplit; ++k)
                if (k < S)
                    in[k] = __ldcg(reinterpret_cast<const float4*>(ws_tile + (static_cast<size_t>(k) * BN + t) * BM) + lane);
            pre = pre_tok<MODE>(tc, t, lane);
        };
        int t = t0 + warp;
        if (t < t1) load(t);
        for (; t < t1; t += kWarps) {
            float4 v = in[0];
#pragma unroll
            for (int k = 1; k < kMaxSplit; ++k)
                if (k < S) {
                    v.x += in[k].x;
                    v.y += in[k].y;
                    v.z += in[k].z;
                    v.w += in[k].w;
                }
            const TokPre cur = pre;
            if (t + kWarps < t1) load(t + kWarps);
            emit_tok<MODE>(tc, t, lane, v, cur);
        }
    }
    __syncthreads();
    if (trace_id >= 0 && trace_id < 512 && threadIdx.x == 0) g_dec_trace[trace_id][3] = dec_gtimer();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

template <int BN, int MODE>
void launch_dec(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int S, int tiles, cudaStream_t st) {
    using C = DecCfg<BN>;
    static bool configured = false;
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_decode_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::kSmem));
        // two CTAs per SM (this kernel and its PDL successor): the full carveout
        SW_CUDA(cudaFuncSetAttribute(gemm_decode_kernel<BN, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(S, tiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    int na = 1;
    if (pdl_mode() && pdl_allowed()) {
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        na = 2;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    SW_CUDA(cudaLaunchKernelEx(&cfg, gemm_decode_kernel<BN, MODE>, a, b, args));
    count_launches(1);
}

template <int BN>
void dispatch_mode(int mode, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int S, int tiles,
                   cudaStream_t st) {
    switch (mode) {
        case EPI_STORE: launch_dec<BN, EPI_STORE>(a, b, args, S, tiles, st); break;
        case EPI_RESID: launch_dec<BN, EPI_RESID>(a, b, args, S, tiles, st); break;
        case EPI_SWIGLU: launch_dec<BN, EPI_SWIGLU>(a, b, args, S, tiles, st); break;
        case EPI_STORE_F32: launch_dec<BN, EPI_STORE_F32>(a, b, args, S, tiles, st); break;
        case EPI_QKV_ROPE: launch_dec<BN, EPI_QKV_ROPE>(a, b, args, S, tiles, st); break;
        default: throw_cuda("gemm_decode: unsupported epilogue", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace

// Split factor from the weight shape and the device only (never the batch, so
// the summation order is the same at every batch size): as many CTAs per tile
// as keep tiles * S within `ctas`, each CTA with >= 2 K-blocks.  A cluster is
// placed inside one GPC, so up to S - 1 CTA slots per GPC can stay unused;
// a grid that only fits the SM count exactly leaves clusters for a second
// wave (Llama-8B QKV: 48 clusters of 6 = 288 of 296 slots).  The budget keeps
// 8 x (S - 1) slots of headroom (B200: 8 GPCs).  (cudaOccupancyMaxActiveClusters is far
// more conservative -- it allowed S = 2 there -- and was 2-5% slower.)
int gemm_decode_splits(int tiles, int nk, int ctas) {
    static const int gpcs = [] {  // SW_DEC_FIT: headroom in GPCs (0 = none)
        const char* v = std::getenv("SW_DEC_FIT");
        return v && *v ? std::atoi(v) : 8;
    }();
    int s = 1;
    while (s < kMaxSplit && tiles * (s + 1) <= ctas - gpcs * s && nk / (s + 1) >= 2) ++s;
    return s;
}

size_t gemm_decode_ws_floats(int tiles, int S, int bn) { return static_cast<size_t>(tiles) * S * bn * BM; }

void gemm_decode_run(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int bn, int S, int tiles,
                     cudaStream_t st) {
    switch (bn) {
        case 32: dispatch_mode<32>(args.mode, a, b, args, S, tiles, st); break;
        case 64: dispatch_mode<64>(args.mode, a, b, args, S, tiles, st); break;
        case 128: dispatch_mode<128>(args.mode, a, b, args, S, tiles, st); break;
        case 256: dispatch_mode<256>(args.mode, a, b, args, S, tiles, st); break;
        default: throw_cuda("gemm_decode: unsupported BN", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace sw

extern "C" int sw_dbg_dec_trace(unsigned long long* host, int n) {
    if (n > 512 * 4) n = 512 * 4;
    return cudaMemcpyFromSymbol(host, sw::g_dec_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}

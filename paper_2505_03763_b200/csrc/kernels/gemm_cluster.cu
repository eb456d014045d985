// Cluster split-K swap-AB GEMM for the decode projections (b <= 64 tokens).
//
// Decode projections have few 128-row weight tiles (Wo/Wd: d/128 = 16 at the
// 1B shape), so one CTA per tile leaves most SMs idle, and a split-K fixup
// through global memory (partials + fence + atomic + a reducing CTA) costs
// more than it saves (profiles/r01/gemm_shapes.txt).  Here a tile is split
// over a thread-block cluster of k CTAs (k <= 8): CTA rank r streams K-blocks
// [r*nk/k, (r+1)*nk/k) into its own TMEM accumulator, parks the fp32 partial
// in its shared memory, and the k partials are reduced through distributed
// shared memory (ld/st.shared::cluster): rank r sums rows [r*128/k, ...) over
// the k ranks in rank order (deterministic) into the leader's buffer; the
// leader runs the fused epilogue (gemm_epilogue.cuh).  ~100 KB of smem per CTA,
// two CTAs per SM.
#include <algorithm>

#include "common.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_sm100.cuh"

namespace sw {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;  // 8 warps: ctl, MMA, 2 producers, 4 epilogue
constexpr int kStages = 4;

template <int BN>
struct ClusterCfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kRingBytes = kStages * kStageBytes;
    static constexpr int kRedBytes = BM * BN * 4;  // one fp32 partial tile
    static_assert(2 * kRedBytes + 128 * 33 * 4 <= kRingBytes, "ring too small for the reduction buffers");
    static constexpr int kTmemCols = BN < 32 ? 32 : BN;
    static constexpr int kSmem = 1024 + kRingBytes + 256 * 16 + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t local_smem, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem), "r"(rank));
    return r;
}
__device__ __forceinline__ float4 ld_dsmem(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t addr, float4 v) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    using C = ClusterCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * C::kABytes;
    // after the main loop the drained ring holds: red (own partial), fin (leader), xchg
    float* red = reinterpret_cast<float*>(smem);
    float* fin = reinterpret_cast<float*>(smem + C::kRedBytes);
    float* xchg = reinterpret_cast<float*>(smem + 2 * C::kRedBytes);
    float* tok_inv = reinterpret_cast<float*>(smem + C::kRingBytes);
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tok_inv) + 256 * 16);
    uint64_t* empty = full + kStages;
    uint64_t* acc_ready = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    griddep_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t k = gridDim.x;          // cluster size (cluster spans x)
    const uint32_t rank = cluster_rank();  // == blockIdx.x
    const int tile = blockIdx.y;
    const int m0 = tile * BM;
    const int nk_total = args.K / BK;
    const int kb0 = static_cast<int>(rank) * nk_total / static_cast<int>(k);
    const int kb1 = static_cast<int>(rank + 1) * nk_total / static_cast<int>(k);
    const int nk = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_ready, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 2 || warp == 3) {
        if (lane == 0) {
            const int p = warp - 2;
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_x = l2_policy_evict_last();
            griddep_wait();  // the activations come from the predecessor kernel
            for (int kb = p; kb < nk; kb += 2) {
                const int s = kb % kStages;
                if (kb >= kStages) mbar_wait(&empty[s], ((kb / kStages) & 1) ^ 1);
                mbar_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], (kb0 + kb) * BK, m0, pol_w);
                tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], (kb0 + kb) * BK, 0, pol_x);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kStages;
                mbar_wait(&full[s], (kb / kStages) & 1);
                tc_fence_after();
                const uint32_t a0 = smem_addr(sA + s * C::kABytes);
                const uint32_t b0 = smem_addr(sB + s * C::kBBytes);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                    umma_bf16(tmem, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                              (kb | kk) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(acc_ready);
        }
        __syncwarp();
    }

    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
    if (warp >= 4) {
        griddep_wait();
        const DecodeFusion& fx = args.fx;
        if (rank == 0) {  // per-token epilogue inputs, gathered while the MMAs run
            for (int t = threadIdx.x - 128; t < BN && t < n_live; t += 128) {
                if (fx.ss_parts) {
                    float ss = 0.f;
                    for (int q = 0; q < fx.ss_nparts; ++q) ss += fx.ss_parts[q * kSsStride + t];
                    tok_inv[t] = rsqrtf(ss / static_cast<float>(fx.norm_dim) + fx.norm_eps);
                }
                if constexpr (MODE == EPI_QKV_ROPE) {
                    const int pos = fx.pos[t];
                    const int page =
                        fx.page_table[static_cast<int64_t>(fx.slot[t]) * fx.max_pages + pos / fx.page_tokens];
                    tok_pos[t] = pos;
                    tok_kv[t] = static_cast<long long>(page) * fx.page_stride +
                                static_cast<long long>(pos % fx.page_tokens) * fx.hd;
                }
            }
        }
        mbar_wait(acc_ready, 0);
        tc_fence_after();
        const uint32_t tb = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t r[32];
        // partial -> own smem, row-major [128][BN] (the ring is drained: all MMAs retired)
        for (int c = 0; c < BN; c += 32) {
            tmem_ld32(tb + c, r);
            tmem_ld_wait();
            float4* dst = reinterpret_cast<float4*>(red + row * BN + c);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        }
        tc_fence_before();
    }
    if (k > 1) {
        cluster_sync_all();  // every rank's partial is in its smem
        // rank r reduces rows [r*128/k, (r+1)*128/k) over the ranks, in rank order
        const int rows_per = BM / static_cast<int>(k);
        const int n4 = rows_per * BN / 4;
        const uint32_t red_local = smem_addr(red + rank * rows_per * BN);
        const uint32_t fin_local = smem_addr(fin + rank * rows_per * BN);
        const uint32_t fin_leader = mapa(fin_local, 0);
        for (int i = threadIdx.x; i < n4; i += kThreads) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (uint32_t q = 0; q < k; ++q) {
                const float4 v = ld_dsmem(mapa(red_local, q) + i * 16);
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            st_dsmem(fin_leader + i * 16, acc);
        }
        cluster_sync_all();  // the leader's fin holds the reduced tile; peers may leave
    }
    if (rank == 0 && warp >= 4) {
        const float* src = k > 1 ? fin : red;
        SwapEpi E{&args, xchg, tok_inv, tok_pos, tok_kv, row, lane, quarter, n_live};
        for (int c = 0; c < BN; c += 32) {
            float v[32];
            const float4* s4 = reinterpret_cast<const float4*>(src + row * BN + c);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float4 t = s4[q];
                v[4 * q] = t.x;
                v[4 * q + 1] = t.y;
                v[4 * q + 2] = t.z;
                v[4 * q + 3] = t.w;
            }
            emit_swap<MODE>(E, m0, c, v);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

template <int BN, int MODE>
void launch_cluster(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int k, int tiles,
                    cudaStream_t st) {
    using C = ClusterCfg<BN>;
    static bool configured = false;
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_cluster_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::kSmem));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(k, tiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = k;
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
    SW_CUDA(cudaLaunchKernelEx(&cfg, gemm_cluster_kernel<BN, MODE>, a, b, args));
    count_launches(1);
}

template <int BN>
void dispatch_mode(int mode, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int k, int tiles,
                   cudaStream_t st) {
    switch (mode) {
        case EPI_STORE: launch_cluster<BN, EPI_STORE>(a, b, args, k, tiles, st); break;
        case EPI_RESID: launch_cluster<BN, EPI_RESID>(a, b, args, k, tiles, st); break;
        case EPI_SWIGLU: launch_cluster<BN, EPI_SWIGLU>(a, b, args, k, tiles, st); break;
        case EPI_STORE_F32: launch_cluster<BN, EPI_STORE_F32>(a, b, args, k, tiles, st); break;
        case EPI_QKV_ROPE: launch_cluster<BN, EPI_QKV_ROPE>(a, b, args, k, tiles, st); break;
        default: throw_cuda("gemm_cluster: unsupported epilogue", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace

// Cluster size from the weight shape only (never the batch): enough CTAs for
// ~two per SM, >= 4 K-blocks each, power of two <= 8.
int gemm_cluster_size(int tiles, int nk, int sms) {
    int k = 1;
    while (k < 8 && tiles * (k * 2) <= 2 * sms && nk / (k * 2) >= 4) k *= 2;
    return k;
}

void gemm_cluster_run(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int bn, int k, int tiles,
                      cudaStream_t st) {
    if (bn == 32) dispatch_mode<32>(args.mode, a, b, args, k, tiles, st);
    else if (bn == 64) dispatch_mode<64>(args.mode, a, b, args, k, tiles, st);
    else throw_cuda("gemm_cluster: BN must be <= 64", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw

#pragma once
// Persistent decode-step kernel for sm_100a: one launch runs a whole decode
// step (all layers + LM head + greedy argmax) on one CTA per SM.
//
// Why: a decode step at b <= 128 rows is a pure weight/KV stream (Llama-1B:
// ~2.5 GB of weights + the KV pages per step), but as 5 kernels per layer it
// pays a launch, a pipeline fill and a drain per projection, and the narrow
// projections (Wo / Wd: d/128 = 16 weight tiles at 1B) cannot spread over
// 148 SMs.  Here every GEMM phase is split stream-K over all CTAs (each CTA
// streams the same number of weight bytes), and the weight producer never
// waits for activations: it runs ahead across phase boundaries into the
// next projection's weights, bounded only by the smem ring, so HBM keeps
// streaming while the CTAs synchronise.
//
// Phases (per layer): QKV (norm-scale + RoPE + paged-KV write epilogue),
// ATTN (split-KV paged attention on the 4 epilogue warps), O (+ residual,
// bf16(x) and sum(x^2) partials), GU (norm-scale + SwiGLU), D (+ residual);
// then the LM head with the packed-argmax epilogue.  Phase p+1 consumes what
// phase p wrote after a grid barrier: every CTA arrives on bar[p] once it has
// finished (or had no work in) phase p; consumers spin on bar[p] == gridDim.
// All CTAs are co-resident (cooperative launch, one CTA per SM by smem).
//
// Warp roles (256 threads):
//   warp 0     barrier init, then the activation producer: TMA of the B
//              operand (BN x 64 box of the phase's input rows) once the
//              producing phase's barrier has completed
//   warp 1     TMEM allocator + tcgen05.mma issuer (one lane)
//   warps 2-3  weight producers: TMA of the A operand (128 x 64 weight box)
//              per (tile, K-block) iteration, interleaved; never wait on the
//              grid barrier
//   warps 4-7  epilogue (TMEM -> fused epilogue) and attention units
// A ring stage's full barrier takes two arrivals (weights + activations) and
// both transactions; the MMA's commit frees it for both producers.
// Split-K partial tiles are reduced by their last contributor, adding the
// partials in CTA order (deterministic, independent of timing and batch).
#include <algorithm>

#include "attn_decode_unit.cuh"
#include "common.cuh"
#include "decode_step.cuh"
#include "gemm_epilogue.cuh"

namespace sw {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;
constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic smem per CTA
constexpr int kContribBatch = 4;  // partials loaded per reduction batch (8 columns each; register bound)

template <int BN, int HD, int G>
struct StepCfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kXchgBytes = 128 * 33 * 4;
    static constexpr int kAttnBytes = attn::decode_unit_smem<HD, G>();
    static constexpr int kUnion = kXchgBytes > kAttnBytes ? kXchgBytes : kAttnBytes;
    static constexpr int kPagesBytes = attn::kMaxChunkPages * 4;
    static constexpr int kTokBytes = 256 * 16;
    static constexpr int kBarBytes = 256;
    static constexpr int kFixed = 1024 + kUnion + kPagesBytes + kTokBytes + kBarBytes;
    static constexpr int kStagesRaw = (kSmemMax - kFixed) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static_assert(kStages >= 3, "stage ring too shallow");
    static constexpr int kSmem = kFixed + kStages * kStageBytes;
    static constexpr int kTmemCols = 2 * BN < 64 ? 64 : 2 * BN;  // two accumulators
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
    while (ld_acquire_gpu(bar) < target) {
    }
}
// generic-proxy writes (epilogue stores) -> async-proxy reads (TMA loads)
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void sync_epi(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

// stream-K schedule of one GEMM phase: (tile, K-block) iterations divided
// evenly over the first min(C, I) CTAs (every participating CTA gets >= 1
// iteration, so a tile's contributors are exactly the owners of its range)
struct PhaseSched {
    int tiles, nk, C, c;
    long long I;
    __device__ void init(int M, int K, int C_, int c_) {
        tiles = M / BM;
        nk = K / BK;
        I = static_cast<long long>(tiles) * nk;
        C = static_cast<int>(min(static_cast<long long>(C_), I));
        c = c_;
    }
    __device__ long long beg(int cc) const { return cc >= C ? I : static_cast<long long>(cc) * I / C; }
    __device__ int owner(long long u) const {  // CTA whose range holds iteration u
        int cc = static_cast<int>((u * C) / I);
        while (cc + 1 < C && beg(cc + 1) <= u) ++cc;
        while (cc > 0 && beg(cc) > u) --cc;
        return cc;
    }
};

struct EpiSmem {
    float* xchg;
    float* tok_inv;
    int* tok_pos;
    long long* tok_kv;
    uint64_t* acc_full;
    uint64_t* acc_empty;
    uint32_t tmem;
};

// Epilogue of one GEMM phase for this CTA's segments (warps 4-7).
template <int BN, int MODE>
__device__ __forceinline__ void epi_gemm(const StepPhase* P, const StepArgs& A, const PhaseSched& sc, int& si,
                                         const EpiSmem& S, int warp, int lane) {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int e = threadIdx.x - 128;
    const GemmArgs& args = P->g;
    const int n_live = min(args.valid_tokens, A.meta->n);
    const DecodeFusion& fx = args.fx;
    for (int t = e; t < BN && t < n_live; t += 128) {
        if (fx.ss_parts) {
            float ss = 0.f;
            for (int q = 0; q < fx.ss_nparts; ++q) ss += __ldcg(fx.ss_parts + q * kSsStride + t);
            S.tok_inv[t] = rsqrtf(ss / static_cast<float>(fx.norm_dim) + fx.norm_eps);
        }
        if constexpr (MODE == EPI_QKV_ROPE) {
            const int pos = fx.pos[t];
            const int page = fx.page_table[static_cast<int64_t>(fx.slot[t]) * fx.max_pages + pos / fx.page_tokens];
            S.tok_pos[t] = pos;
            S.tok_kv[t] = static_cast<long long>(page) * fx.page_stride + static_cast<long long>(pos % fx.page_tokens) * fx.hd;
        }
    }
    sync_epi(1);
    SwapEpi E{&args, S.xchg, S.tok_inv, S.tok_pos, S.tok_kv, row, lane, quarter, n_live};
    uint32_t r[32];
    int pending[2];  // partial tiles of this CTA (its first and last segment)
    int n_pending = 0;
    const long long end = sc.beg(sc.c + 1);
    for (long long u = sc.beg(sc.c); u < end;) {
        const int tile = static_cast<int>(u / sc.nk);
        const long long t0 = static_cast<long long>(tile) * sc.nk;
        const long long stop = min(end, t0 + sc.nk);
        const bool whole = u == t0 && stop == t0 + sc.nk;
        u = stop;
        const int a = si & 1;
        mbar_wait(&S.acc_full[a], (si >> 1) & 1);
        tc_fence_after();
        ++si;
        const uint32_t tb = S.tmem + a * BN + (static_cast<uint32_t>(quarter * 32) << 16);
        const int m0 = tile * BM;
        auto release_acc = [&] {
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.acc_empty[a]);
        };
        if (whole) {
            for (int c = 0; c < BN; c += 32) {
                tmem_ld32(tb + c, r);
                tmem_ld_wait();
                if (c == BN - 32) release_acc();
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                emit_swap<MODE>(E, m0, c, v);
            }
            continue;
        }
        // partial tile: park it and count it in (never wait here: a CTA's first
        // segment shares its tile with the previous CTA's LAST segment)
        const int slot = sc.beg(sc.c) >= t0 ? 0 : 1;  // the CTA's first or last segment
        float* part = A.ws + (static_cast<size_t>(sc.c) * 2 + slot) * BN * 128;
        for (int c = 0; c < BN; c += 32) {
            tmem_ld32(tb + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float4* dst = reinterpret_cast<float4*>(part + ((static_cast<size_t>(c / 8 + q) * 128 + row) * 8));
                __stcg(dst, make_float4(__uint_as_float(r[8 * q]), __uint_as_float(r[8 * q + 1]),
                                        __uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3])));
                __stcg(dst + 1, make_float4(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]),
                                            __uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7])));
            }
        }
        release_acc();
        sync_epi(2);
        if (e == 0) {
            __threadfence();
            atomicAdd(A.counters + P->cnt_off + tile, 1u);
        }
        pending[n_pending++] = tile;
    }
    // Reduce the partial tiles this CTA contributed to, together with their
    // other contributors: contributor j sums 8-token column groups j, j + ncon,
    // ... over all parked partials in CTA order (deterministic) and runs the
    // epilogue on them.
    for (int pi = 0; pi < n_pending; ++pi) {
        const int tile = pending[pi];
        const long long t0 = static_cast<long long>(tile) * sc.nk;
        const int c_first = sc.owner(t0), c_last = sc.owner(t0 + sc.nk - 1);
        const int ncon = c_last - c_first + 1;
        if (e == 0) grid_wait(A.counters + P->cnt_off + tile, static_cast<unsigned>(ncon));  // all parked
        sync_epi(2);
        const int m0 = tile * BM;
        const int groups = min(BN, n_live + 7) / 8;
        const int g0 = A.debug_single_reducer ? (sc.c == c_first ? 0 : groups) : sc.c - c_first;
        const int gstep = A.debug_single_reducer ? 1 : ncon;
        for (int gidx = g0; gidx < groups; gidx += gstep) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int k0 = 0; k0 < ncon; k0 += kContribBatch) {
                float4 lo[kContribBatch], hi[kContribBatch];
#pragma unroll
                for (int k = 0; k < kContribBatch; ++k) {
                    if (k0 + k < ncon) {
                        const int cc = c_first + k0 + k;
                        const int sl = sc.beg(cc) >= t0 ? 0 : 1;
                        const float4* pp = reinterpret_cast<const float4*>(
                            A.ws + (static_cast<size_t>(cc) * 2 + sl) * BN * 128 + (static_cast<size_t>(gidx) * 128 + row) * 8);
                        lo[k] = __ldcg(pp);
                        hi[k] = __ldcg(pp + 1);
                    }
                }
#pragma unroll
                for (int k = 0; k < kContribBatch; ++k) {  // contributor (CTA) order: deterministic
                    if (k0 + k < ncon) {
                        acc[0] += lo[k].x; acc[1] += lo[k].y; acc[2] += lo[k].z; acc[3] += lo[k].w;
                        acc[4] += hi[k].x; acc[5] += hi[k].y; acc[6] += hi[k].z; acc[7] += hi[k].w;
                    }
                }
            }
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = j < 8 ? acc[j & 7] : 0.f;
            emit_swap<MODE>(E, m0, gidx * 8, v, 8);
        }
    }
}

template <int BN, int HD, int G>
__global__ void __launch_bounds__(kThreads, 1) decode_step_kernel(const __grid_constant__ StepArgs A) {
    using Cf = StepCfg<BN, HD, G>;
    constexpr int S = Cf::kStages;
    constexpr int KB = attn::decode_kb<HD>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = sA + S * Cf::kABytes;
    uint8_t* uni = sB + S * Cf::kBBytes;  // GEMM epilogue exchange | attention buffers
    int32_t* s_pages = reinterpret_cast<int32_t*>(uni + Cf::kUnion);
    float* tok_inv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s_pages) + Cf::kPagesBytes);
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tok_inv) + Cf::kTokBytes);
    uint64_t* empty = full + S;
    uint64_t* acc_full = empty + S;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    uint32_t* attn_last = tmem_slot + 1;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int C = gridDim.x, c = blockIdx.x;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 2);  // weights + activations
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);  // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, Cf::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 2 || warp == 3) {
        // ------------------------------------------------ weight producers
        if (lane == 0) {
            const int p = warp - 2;
            const uint64_t pol_w = l2_policy_evict_first();
            long long gi = 0;
            for (int ph = 0; ph < A.n_phases; ++ph) {
                const StepPhase* P = A.phases + ph;
                if (P->kind != PHASE_GEMM) continue;
                PhaseSched sc;
                sc.init(P->M, P->K, C, c);
                const CUtensorMap* tm = A.maps + P->w_map;
                const long long b = sc.beg(c), e = sc.beg(c + 1);
                for (long long u = b; u < e; ++u, ++gi) {
                    if ((gi & 1) != p) continue;
                    const int tile = static_cast<int>(u / sc.nk);
                    const int kb = static_cast<int>(u - static_cast<long long>(tile) * sc.nk);
                    const int s = static_cast<int>(gi % S);
                    mbar_wait(&empty[s], static_cast<uint32_t>(((gi / S) & 1) ^ 1));
                    if (A.trace && p == 0) {
                        unsigned long long* tr = A.trace + (static_cast<size_t>(ph) * C + c) * 8;
                        if (u == b) tr[4] = globaltimer_ns();
                        if (u + 2 >= e) tr[5] = globaltimer_ns();
                    }
                    mbar_expect_tx(&full[s], Cf::kABytes);
                    tma_load_2d(sA + s * Cf::kABytes, tm, &full[s], kb * BK, tile * BM, pol_w);
                }
            }
        }
        __syncwarp();
    } else if (warp == 0) {
        // ------------------------------------------------ activation producer
        if (lane == 0) {
            const uint64_t pol_x = l2_policy_evict_last();
            long long gi = 0;
            for (int ph = 0; ph < A.n_phases; ++ph) {
                const StepPhase* P = A.phases + ph;
                if (P->kind != PHASE_GEMM) continue;
                PhaseSched sc;
                sc.init(P->M, P->K, C, c);
                const long long b = sc.beg(c), e = sc.beg(c + 1);
                if (b >= e) continue;
                if (ph > 0) {
                    grid_wait(A.bar + ph - 1, static_cast<unsigned>(C));  // the producing phase is done
                    fence_proxy_async_global();
                }
                if (A.trace) A.trace[(static_cast<size_t>(ph) * C + c) * 8 + 3] = globaltimer_ns();
                const CUtensorMap* tm = A.maps + P->x_map;
                for (long long u = b; u < e; ++u, ++gi) {
                    const int kb = static_cast<int>(u % sc.nk);
                    const int s = static_cast<int>(gi % S);
                    mbar_wait(&empty[s], static_cast<uint32_t>(((gi / S) & 1) ^ 1));
                    mbar_expect_tx(&full[s], Cf::kBBytes);
                    tma_load_2d(sB + s * Cf::kBBytes, tm, &full[s], kb * BK, 0, pol_x);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            long long gi = 0;
            int si = 0;
            for (int ph = 0; ph < A.n_phases; ++ph) {
                const StepPhase* P = A.phases + ph;
                if (P->kind != PHASE_GEMM) continue;
                PhaseSched sc;
                sc.init(P->M, P->K, C, c);
                const long long e = sc.beg(c + 1);
                for (long long u = sc.beg(c); u < e;) {
                    const long long seg0 = u;
                    const long long stop = min(e, (u / sc.nk + 1) * sc.nk);
                    const int a = si & 1;
                    mbar_wait(&acc_empty[a], static_cast<uint32_t>(((si >> 1) & 1) ^ 1));
                    tc_fence_after();
                    const uint32_t acc = tmem + a * BN;
                    for (; u < stop; ++u, ++gi) {
                        const int s = static_cast<int>(gi % S);
                        mbar_wait(&full[s], static_cast<uint32_t>((gi / S) & 1));
                        tc_fence_after();
                        if (A.trace) {
                            unsigned long long* tr = A.trace + (static_cast<size_t>(ph) * C + c) * 8;
                            if (u == sc.beg(c)) tr[6] = globaltimer_ns();
                            if (u + 1 == e) tr[7] = globaltimer_ns();
                        }
                        const uint32_t a0 = smem_addr(sA + s * Cf::kABytes);
                        const uint32_t b0 = smem_addr(sB + s * Cf::kBBytes);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            umma_bf16(acc, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                                      (u > seg0 || k > 0) ? 1u : 0u);
                        umma_commit(&empty[s]);
                    }
                    umma_commit(&acc_full[a]);
                    ++si;
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue + attention
        const int e = threadIdx.x - 128;
        EpiSmem es{reinterpret_cast<float*>(uni), tok_inv, tok_pos, tok_kv, acc_full, acc_empty, tmem};
        int si = 0;
        for (int ph = 0; ph < A.n_phases; ++ph) {
            const StepPhase* P = A.phases + ph;
            const int kind = P->kind;
            PhaseSched sc;
            bool has = true;
            if (kind == PHASE_GEMM) {
                sc.init(P->M, P->K, C, c);
                has = sc.beg(c) < sc.beg(c + 1);
            }
            if (A.trace && e == 0) A.trace[(static_cast<size_t>(ph) * C + c) * 8 + 0] = globaltimer_ns();
            if (has) {
                if (ph > 0) {
                    if (e == 0) grid_wait(A.bar + ph - 1, static_cast<unsigned>(C));
                    sync_epi(3);
                }
                if (A.trace && e == 0) A.trace[(static_cast<size_t>(ph) * C + c) * 8 + 1] = globaltimer_ns();
                if (kind == PHASE_GEMM) {
                    switch (P->mode) {
                        case EPI_QKV_ROPE: epi_gemm<BN, EPI_QKV_ROPE>(P, A, sc, si, es, warp, lane); break;
                        case EPI_RESID: epi_gemm<BN, EPI_RESID>(P, A, sc, si, es, warp, lane); break;
                        case EPI_SWIGLU: epi_gemm<BN, EPI_SWIGLU>(P, A, sc, si, es, warp, lane); break;
                        case EPI_ARGMAX: epi_gemm<BN, EPI_ARGMAX>(P, A, sc, si, es, warp, lane); break;
                        default: epi_gemm<BN, EPI_STORE>(P, A, sc, si, es, warp, lane); break;
                    }
                } else {
                    const DecodeAttnArgs& at = A.attn;
                    const int n = A.meta->n;
                    const int want = cdiv(A.attn_target, n * at.Hkv);
                    const int cap = min(at.max_splits, max(want, cdiv(at.max_ctx, attn::kMaxChunkPages * attn::kPage)));
                    const int per_pair = min(want, cap);
                    const int total = n * at.Hkv * per_pair;
                    for (int u = c; u < total; u += C) {
                        const int pair = u / per_pair, split = u - pair * per_pair;
                        const int row = pair / at.Hkv, hk = pair - row * at.Hkv;
                        const int ctx = A.meta->pos[row] + 1;
                        const attn::SplitPlan plan = attn::decode_split_plan<KB>(ctx, want, per_pair);
                        if (split >= plan.splits) continue;
                        attn::decode_unit<HD, G, KB>(at, P->q, P->kv, P->out, row, hk, split, plan, ctx, uni, s_pages,
                                                     attn_last, e, [] { sync_epi(3); });
                    }
                }
            }
            // phase done for this CTA (stores issued by all 128 threads)
            fence_proxy_async_global();
            sync_epi(3);
            if (e == 0) {
                if (A.trace) A.trace[(static_cast<size_t>(ph) * C + c) * 8 + 2] = globaltimer_ns();
                __threadfence();
                atomicAdd(A.bar + ph, 1u);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, Cf::kTmemCols);
    }
}

template <int BN, int HD, int G>
void launch_step(const StepArgs& a, int ctas, cudaStream_t st) {
    using Cf = StepCfg<BN, HD, G>;
    static bool configured = false;
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(decode_step_kernel<BN, HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Cf::kSmem));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cf::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barriers rely on it
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SW_CUDA(cudaLaunchKernelEx(&cfg, decode_step_kernel<BN, HD, G>, a));
    count_launches(1);
}

template <int HD, int G>
inline void dispatch_bn(const StepArgs& a, int bn, int ctas, cudaStream_t st) {
    switch (bn) {
        case 32: launch_step<32, HD, G>(a, ctas, st); break;
        case 64: launch_step<64, HD, G>(a, ctas, st); break;
        case 128: launch_step<128, HD, G>(a, ctas, st); break;
        default: throw_cuda("decode_step: unsupported row tile", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

template <int HD, int G>
int stages_bn(int bn) {
    switch (bn) {
        case 32: return StepCfg<32, HD, G>::kStages;
        case 64: return StepCfg<64, HD, G>::kStages;
        case 128: return StepCfg<128, HD, G>::kStages;
        default: return 0;
    }
}

}  // namespace

// one (head_dim, group) configuration per translation unit (parallel build)
#define SW_DECODE_STEP_INSTANTIATE(HD_, G_)                                                         \
    void decode_step_launch_##HD_##_##G_(const StepArgs& a, int bn, int ctas, cudaStream_t st) {    \
        dispatch_bn<HD_, G_>(a, bn, ctas, st);                                                      \
    }                                                                                               \
    int decode_step_stages_##HD_##_##G_(int bn) { return stages_bn<HD_, G_>(bn); }

}  // namespace sw

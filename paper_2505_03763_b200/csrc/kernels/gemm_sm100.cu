// tcgen05/TMEM GEMM for sm_100a with fused epilogues -- the tensor-core core
// of both phases.
//
//   Y[t, f] = sum_k X[t, k] * W[f, k]      X: activations bf16 [T, K]
//                                          W: weights     bf16 [F, K]
// Prefill ("normal"):  A = X (UMMA M = 128 tokens), B = W (UMMA N = BN features)
// Decode  ("swap-AB"): A = W (UMMA M = 128 features), B = X (UMMA N = BN >= b
//                      tokens, TMA pads).  The weight stream is the A operand,
//                      so a batch of b <= 256 rows costs one pass over W.
//
// One CTA = one 128 x BN output tile, 6 warps:
//   warp 0  TMA producer (one lane): A/B K-blocks of 64 into a STAGES-deep
//           ring of 128B-swizzled smem, completion by mbarrier tx-count;
//   warp 1  TMEM allocator + MMA issuer (one lane): 4 x tcgen05.mma
//           (128 x BN x 16) per K-block, tcgen05.commit frees the ring slot;
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 (warp%4 picks its 32 TMEM
//           lanes) -> registers -> fused epilogue -> global.
// Epilogues: STORE (bf16), RESID (fp32 residual +=), SWIGLU over
// [gate 64 | up 64] feature blocks (bf16 out, half width), ARGMAX (packed
// 64-bit atomicMax per token: LM head + greedy sampling in one pass).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "gemm_sm100.cuh"

namespace sw {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;

template <int BN, bool SWAP, bool SMALL = false>
struct GemmCfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    // SMALL: ~100 KB so two CTAs stream weights per SM
    static constexpr int kBudget = (SMALL && BN <= 64) ? 100 * 1024 : 200 * 1024;
    static constexpr int kStagesRaw = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
    static constexpr int kStages = kStagesRaw >= 8 ? 8 : 4;  // multiple of the 4 producer warps
    static_assert(kStagesRaw >= 4, "smem budget below 4 stages");
    static constexpr int kTmemCols = BN < 32 ? 32 : BN;
    // epilogue exchanges (SwiGLU / RoPE pairs, 128 x 33 fp32) reuse the drained stage ring
    static_assert(kStages * kStageBytes >= 128 * 33 * 4, "stage ring too small for the exchange buffer");
    static constexpr int kTokInfoBytes = 256 * 16;  // per-token 1/rms, position, KV offset (decode)
    static constexpr int kSmem = 1024 + kStages * kStageBytes + kTokInfoBytes + 256;
};

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.0f + __expf(-g)) * u; }

template <int BN, int MODE, bool SWAP, bool SMALL>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    using C = GemmCfg<BN, SWAP, SMALL>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kABytes;
    float* xchg = reinterpret_cast<float*>(sA);  // epilogue only: the ring is drained by then
    float* tok_inv = reinterpret_cast<float*>(sB + C::kStages * C::kBBytes);  // [256]
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);                       // [256]
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);            // [256]
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tok_inv) + C::kTokInfoBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* acc_ready = empty + C::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_ready + 1);

    griddep_launch_dependents();  // let the next kernel of the step start its prologue
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    // split-K: this CTA owns K-blocks [kb0, kb1)
    const int nk_total = args.K / BK;
    const int kb0 = static_cast<int>(blockIdx.z) * nk_total / static_cast<int>(gridDim.z);
    const int kb1 = (static_cast<int>(blockIdx.z) + 1) * nk_total / static_cast<int>(gridDim.z);
    const int nk = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_ready, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch_desc(&tmA);
            tma_prefetch_desc(&tmB);
        }
        __syncwarp();
    } else if (warp >= 2) {
        // ---------------------------------------------------------- producers
        // One issuing thread completes only ~1 bulk copy per ~600 cycles
        // (tools/tma_bench2.cu), so the four epilogue warps share the K loop:
        // warp p issues K-blocks kb = p, p+4, ... (stages s = kb % S, S % 4 == 0,
        // so each stage has one owner), then turns into an epilogue warp.
        if (lane == 0) {
            // Weights are streamed once per launch (evict-first); activations
            // are re-read by every feature tile (evict-last).
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_x = l2_policy_evict_last();
            const uint64_t pol_a = SWAP ? pol_w : pol_x;
            const uint64_t pol_b = SWAP ? pol_x : pol_w;
            // Tiles start their K walk at staggered offsets so the CTAs of a
            // one-wave launch do not stream in lockstep.
            const int rot = args.stagger ? static_cast<int>((blockIdx.y * 7u + blockIdx.x * 3u) % nk) : 0;
            auto kidx = [&](int kb) {
                const int kk = kb + rot;
                return kb0 + (kk >= nk ? kk - nk : kk);
            };
            // The first ring fill of the constant operand (decode: the weights)
            // is issued before waiting on the predecessor kernel (PDL), so the
            // weight stream starts while the previous kernel drains.
            const uint8_t* pre_dst = SWAP ? sA : sB;
            const int pre_bytes = SWAP ? C::kABytes : C::kBBytes;
            const void* pre_map = SWAP ? static_cast<const void*>(&tmA) : static_cast<const void*>(&tmB);
            const int pre_row = SWAP ? m0 : n0;
            const uint64_t pre_pol = pol_w;
            for (int kb = warp - 2; kb < nk && kb < C::kStages; kb += 4) {
                const int s = kb % C::kStages;
                mbar_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(const_cast<uint8_t*>(pre_dst) + s * pre_bytes, pre_map, &full[s], kidx(kb) * BK, pre_row,
                            pre_pol);
            }
            griddep_wait();
            for (int kb = warp - 2; kb < nk; kb += 4) {
                const int s = kb % C::kStages;
                const uint32_t ph = (kb / C::kStages) & 1;
                const int kc = kidx(kb) * BK;
                if (kb < C::kStages) {  // weights already in flight: the activation half
                    if (SWAP) tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], kc, n0, pol_b);
                    else tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], kc, m0, pol_a);
                    continue;
                }
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], C::kStageBytes);
                tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], kc, m0, pol_a);
                tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], kc, n0, pol_b);
            }
        }
        __syncwarp();
        griddep_wait();  // every epilogue thread reads predecessor outputs below
    }
    if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % C::kStages;
                const uint32_t ph = (kb / C::kStages) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a0 = smem_addr(sA + s * C::kABytes);
                const uint32_t b0 = smem_addr(sB + s * C::kBBytes);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                              (kb | k) != 0);
                umma_commit(&empty[s]);
            }
            umma_commit(acc_ready);
        }
        __syncwarp();
    }
    if (warp >= 2) {
        // ------------------------------------------------------------ epilogue
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
        const int row = quarter * 32 + lane;  // accumulator row inside the tile
        if constexpr (SWAP) {
            // per-token epilogue inputs, gathered while the MMAs still run
            const DecodeFusion& fx = args.fx;
            const int nl = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
            for (int t = threadIdx.x - 64; t < BN && n0 + t < nl; t += 128) {
                const int tg = n0 + t;
                if (fx.ss_parts) {
                    float ss = 0.f;
                    for (int p = 0; p < fx.ss_nparts; ++p) ss += fx.ss_parts[p * kSsStride + tg];
                    tok_inv[t] = rsqrtf(ss / static_cast<float>(fx.norm_dim) + fx.norm_eps);
                }
                if constexpr (MODE == EPI_QKV_ROPE) {
                    const int pos = fx.pos[tg];
                    const int page = fx.page_table[static_cast<int64_t>(fx.slot[tg]) * fx.max_pages + pos / fx.page_tokens];
                    tok_pos[t] = pos;
                    tok_kv[t] = static_cast<long long>(page) * fx.page_stride +
                                static_cast<long long>(pos % fx.page_tokens) * fx.hd;
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        mbar_wait(acc_ready, 0);
        tc_fence_after();
        const uint32_t tbase = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t r[32];
        const int n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        if constexpr (!SWAP) {
            // row = token, columns = features
            const int t = m0 + row;
            const bool live = t < n_live;
            if constexpr (MODE == EPI_SWIGLU) {
                for (int blk = 0; blk < BN / 128; ++blk) {
#pragma unroll
                    for (int half = 0; half < 64; half += 32) {
                        uint32_t u[32];
                        tmem_ld32(tbase + blk * 128 + half, r);
                        tmem_ld32(tbase + blk * 128 + 64 + half, u);
                        tmem_ld_wait();
                        if (live) {
                            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(args.out) +
                                                 static_cast<size_t>(t) * args.ldo + (n0 + blk * 128) / 2 + half;
                            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                uint4 v;
                                v.x = pack_bf2(silu_mul(__uint_as_float(r[8 * q + 0]), __uint_as_float(u[8 * q + 0])),
                                               silu_mul(__uint_as_float(r[8 * q + 1]), __uint_as_float(u[8 * q + 1])));
                                v.y = pack_bf2(silu_mul(__uint_as_float(r[8 * q + 2]), __uint_as_float(u[8 * q + 2])),
                                               silu_mul(__uint_as_float(r[8 * q + 3]), __uint_as_float(u[8 * q + 3])));
                                v.z = pack_bf2(silu_mul(__uint_as_float(r[8 * q + 4]), __uint_as_float(u[8 * q + 4])),
                                               silu_mul(__uint_as_float(r[8 * q + 5]), __uint_as_float(u[8 * q + 5])));
                                v.w = pack_bf2(silu_mul(__uint_as_float(r[8 * q + 6]), __uint_as_float(u[8 * q + 6])),
                                               silu_mul(__uint_as_float(r[8 * q + 7]), __uint_as_float(u[8 * q + 7])));
                                d4[q] = v;
                            }
                        }
                    }
                }
            } else {
                for (int c = 0; c < BN; c += 32) {
                    tmem_ld32(tbase + c, r);
                    tmem_ld_wait();
                    if (!live) continue;
                    if constexpr (MODE == EPI_STORE) {
                        uint4* d4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.out) +
                                                             static_cast<size_t>(t) * args.ldo + n0 + c);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint4 v;
                            v.x = pack_bf2(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1]));
                            v.y = pack_bf2(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3]));
                            v.z = pack_bf2(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]));
                            v.w = pack_bf2(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7]));
                            d4[q] = v;
                        }
                    } else if constexpr (MODE == EPI_STORE_F32) {
                        float4* d4 = reinterpret_cast<float4*>(static_cast<float*>(args.out) +
                                                               static_cast<size_t>(t) * args.ldo + n0 + c);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            d4[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                    } else if constexpr (MODE == EPI_RESID) {
                        // all loads first, then all stores: 8 independent requests in
                        // flight instead of 8 serialised read-modify-write round trips
                        float4* d4 = reinterpret_cast<float4*>(static_cast<float*>(args.out) +
                                                               static_cast<size_t>(t) * args.ldo + n0 + c);
                        float4 old[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) old[q] = __ldcg(d4 + q);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            old[q].x += __uint_as_float(r[4 * q + 0]);
                            old[q].y += __uint_as_float(r[4 * q + 1]);
                            old[q].z += __uint_as_float(r[4 * q + 2]);
                            old[q].w += __uint_as_float(r[4 * q + 3]);
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) d4[q] = old[q];
                    }
                }
            }
        } else {
            // row = feature (weight row), columns = tokens
            const int f = m0 + row;
            const DecodeFusion& fx = args.fx;
            // 32 fp32 values per lane -> lane j holds the sum over the warp of value j (31 shuffles)
            auto transpose_sum = [&](float (&v)[32]) {
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const bool upper = (lane & off) != 0;
#pragma unroll
                    for (int i = 0; i < off; ++i) {
                        const float send = upper ? v[i] : v[i + off];
                        const float keep = upper ? v[i + off] : v[i];
                        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                    }
                }
            };
            auto emit = [&](int c, const uint32_t (&raw)[32]) {
                const int tcount = min(32, n_live - (n0 + c));
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
                if (fx.ss_parts && MODE != EPI_RESID) {  // RMSNorm of the input rows, folded in
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < tcount) v[j] *= tok_inv[c + j];
                }
                if constexpr (MODE == EPI_STORE) {
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                        static_cast<__nv_bfloat16*>(args.out)[static_cast<size_t>(n0 + c + j) * args.ldo + f] =
                            __float2bfloat16_rn(v[j]);
                } else if constexpr (MODE == EPI_STORE_F32) {
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                        static_cast<float*>(args.out)[static_cast<size_t>(n0 + c + j) * args.ldo + f] = v[j];
                } else if constexpr (MODE == EPI_RESID) {
                    float* col = static_cast<float*>(args.out) + static_cast<size_t>(n0 + c) * args.ldo + f;
                    float x[32];
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) x[j] =
                        j < tcount ? __ldcg(col + static_cast<size_t>(j) * args.ldo) : 0.f;
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) {
                        x[j] += v[j];
                        if (j < tcount) {
                            col[static_cast<size_t>(j) * args.ldo] = x[j];
                            if (fx.x_bf16)
                                fx.x_bf16[static_cast<size_t>(n0 + c + j) * args.ldo + f] = __float2bfloat16_rn(x[j]);
                        }
                        x[j] = j < tcount ? x[j] * x[j] : 0.f;
                    }
                    if (fx.ss_part_out) {  // this tile's sum(x^2) per token, for the next RMSNorm
                        transpose_sum(x);  // lane j: the warp's partial for token c + j
                        xchg[quarter * 32 + lane] = x[0];
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                        if (quarter == 0 && lane < tcount)  // fixed order over the 4 warps: deterministic
                            fx.ss_part_out[static_cast<size_t>(blockIdx.y) * kSsStride + n0 + c + lane] =
                                (xchg[lane] + xchg[32 + lane]) + (xchg[64 + lane] + xchg[96 + lane]);
                        asm volatile("bar.sync 1, 128;" ::: "memory");
                    }
                } else if constexpr (MODE == EPI_SWIGLU) {
                    // lanes 0-63 of the tile hold gate rows, 64-127 the matching up rows
                    if (row >= 64) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) xchg[(row - 64) * 33 + j] = v[j];
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (row < 64) {
                        const int g = m0 / 2 + row;
                        _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                            static_cast<__nv_bfloat16*>(args.out)[static_cast<size_t>(n0 + c + j) * args.ldo + g] =
                                __float2bfloat16_rn(silu_mul(v[j], xchg[row * 33 + j]));
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                } else if constexpr (MODE == EPI_ARGMAX) {
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount) {
                        unsigned long long key = argmax_key(v[j], static_cast<uint32_t>(args.feature_offset + f));
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                            key = other > key ? other : key;
                        }
                        if (lane == 0) atomicMax(args.argmax + n0 + c + j, key);
                    }
                } else if constexpr (MODE == EPI_QKV_ROPE) {
                    // rotate-half RoPE: row r pairs with r ^ (hd/2) inside its head
                    const int hd = fx.hd, half = hd >> 1;
                    const int head = f / hd, i = f % hd;
#pragma unroll
                    for (int j = 0; j < 32; ++j) xchg[row * 33 + j] = v[j];
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    const int prow = row ^ half;
                    const bool is_v = head >= fx.H + fx.Hkv;
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) {
                        if (j >= tcount) continue;
                        const int t = n0 + c + j;
                        const int pos = tok_pos[c + j];
                        float out = v[j];
                        if (!is_v) {
                            const float2 cs = fx.rope_cs[static_cast<int64_t>(pos) * half + (i & (half - 1))];
                            const float b = xchg[prow * 33 + j];
                            out = i < half ? v[j] * cs.x - b * cs.y : v[j] * cs.x + b * cs.y;
                        }
                        if (head < fx.H) {
                            fx.q_out[static_cast<size_t>(t) * fx.H * hd + f] = __float2bfloat16_rn(out);
                        } else {
                            const int kvh = is_v ? head - fx.H - fx.Hkv : head - fx.H;
                            __nv_bfloat16* dst = fx.kv_layer + tok_kv[c + j] + (is_v ? fx.page_stride / 2 : 0) +
                                                 static_cast<int64_t>(kvh) * fx.page_tokens * hd + i;
                            *dst = __float2bfloat16_rn(out);
                        }
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
            };
            if (gridDim.z == 1) {
                for (int c = 0; c < BN; c += 32) {
                    tmem_ld32(tbase + c, r);
                    tmem_ld_wait();
                    emit(c, r);
                }
            } else {
                // Split-K: park this CTA's fp32 partial tile in the (L2-resident)
                // workspace; the last CTA of the tile to finish reduces all
                // partials in split order (deterministic) and runs the epilogue.
                const int tile = blockIdx.y * gridDim.x + blockIdx.x;
                const int splits = gridDim.z;
                float* part = args.ws + static_cast<size_t>(tile) * splits * BN * 128;
                for (int c = 0; c < BN; c += 32) {
                    tmem_ld32(tbase + c, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        __stcg(part + (static_cast<size_t>(blockIdx.z) * BN + c + j) * 128 + row, __uint_as_float(r[j]));
                }
                __threadfence();
                asm volatile("bar.sync 2, 128;" ::: "memory");
                uint32_t* last_flag = reinterpret_cast<uint32_t*>(tmem_slot + 1);
                if (threadIdx.x == 64) {
                    const unsigned prev = atomicAdd(args.counters + tile, 1u);
                    *last_flag = prev == static_cast<unsigned>(splits - 1);
                }
                asm volatile("bar.sync 2, 128;" ::: "memory");
                if (*last_flag) {
                    __threadfence();
                    for (int c = 0; c < BN; c += 32) {
                        float acc[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
#pragma unroll 4
                        for (int z = 0; z < splits; ++z)
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                acc[j] += __ldcg(part + (static_cast<size_t>(z) * BN + c + j) * 128 + row);
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(acc[j]);
                        emit(c, r);
                    }
                    if (threadIdx.x == 64) args.counters[tile] = 0u;  // re-arm for the next launch
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

// ---------------------------------------------------------------- host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        SW_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw_cuda("cuTensorMapEncodeTiled lookup", cudaErrorUnknown, __FILE__, __LINE__);
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

template <int BN, int MODE, bool SWAP, bool SMALL>
void launch_cfg(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, cudaStream_t st) {
    using C = GemmCfg<BN, SWAP, SMALL>;
    static bool configured = false;  // per instantiation
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, MODE, SWAP, SMALL>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        configured = true;
    }
    dim3 grid(args.N / BN, cdiv(args.M, BM), args.splits > 0 ? args.splits : 1);
    launch_k(gemm_tc_kernel<BN, MODE, SWAP, SMALL>, grid, dim3(kThreads), C::kSmem, st, a, b, args);
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

template <int BN, int MODE, bool SWAP>
void launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, cudaStream_t st) {
    // decode (swap) tiles with BN <= 64 default to the two-CTAs-per-SM budget;
    // SW_GEMM_SMALL=0/1 overrides (tuning sweeps)
    static const int small_env = env_int("SW_GEMM_SMALL", -1);
    const bool small = small_env >= 0 ? small_env != 0 : (SWAP && BN <= 64);
    if (small) launch_cfg<BN, MODE, SWAP, true>(a, b, args, st);
    else launch_cfg<BN, MODE, SWAP, false>(a, b, args, st);
}

template <bool SWAP, int MODE>
void dispatch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, cudaStream_t st) {
    switch (bn) {
        case 32: launch_one<32, MODE, SWAP>(a, b, args, st); break;
        case 64: launch_one<64, MODE, SWAP>(a, b, args, st); break;
        case 128: launch_one<128, MODE, SWAP>(a, b, args, st); break;
        case 256: launch_one<256, MODE, SWAP>(a, b, args, st); break;
        default: throw_cuda("gemm: unsupported BN", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace

CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_cuda("cuTensorMapEncodeTiled", cudaErrorInvalidValue, __FILE__, __LINE__);
    return m;
}

const CUtensorMap& tmap_cached(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, uint64_t, uint64_t, uint32_t>, CUtensorMap> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(base, rows, cols, box_rows);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, make_tmap_bf16(base, rows, cols, box_rows)).first;
    return it->second;
}

int gemm_pick_bn_swap(int tokens) {
    if (tokens <= 32) return 32;
    if (tokens <= 64) return 64;
    if (tokens <= 128) return 128;
    return 256;
}

void gemm_run(const GemmProblem& p, cudaStream_t st) {
    if (p.K % BK != 0) throw_cuda("gemm: K must be a multiple of 64", cudaErrorInvalidValue, __FILE__, __LINE__);
    GemmArgs a{};
    a.K = p.K;
    a.mode = p.mode;
    a.out = p.out;
    a.ldo = p.ldo;
    a.argmax = p.argmax;
    a.feature_offset = p.feature_offset;
    a.valid_tokens = p.tokens;
    a.live_tokens = p.live_tokens;
    a.splits = 1;
    a.fx = p.fx;
    a.ws = p.ws;
    a.counters = p.counters;
    if (p.swap) {
        // split-K from the weight shape only (never the batch), so results are
        // identical for every batch size: ~2 CTAs per SM of weight streams,
        // >= 4 K-blocks per split.
        if (p.ws && p.counters && p.mode != EPI_ARGMAX) {
            const int tiles = p.features / BM, nk = p.K / BK;
            int sp = std::max(1, 296 / tiles);
            sp = std::min(sp, nk / 4);
            sp = std::min(sp, 16);
            static const int forced = env_int("SW_GEMM_SPLITS", 0);  // tuning override
            if (forced > 0) sp = std::min(forced, nk);
            a.splits = std::max(sp, 1);
            if (static_cast<size_t>(tiles) * a.splits * 256 * 128 > p.ws_floats || tiles > p.n_counters) a.splits = 1;
        }
        if (p.features % BM != 0)
            throw_cuda("gemm(swap): feature count must be a multiple of 128", cudaErrorInvalidValue, __FILE__, __LINE__);
        if (p.tokens > 256) throw_cuda("gemm(swap): at most 256 tokens", cudaErrorInvalidValue, __FILE__, __LINE__);
        const int bn = gemm_pick_bn_swap(p.tokens);
        a.M = p.features;
        a.N = bn;
        static const int stagger = env_int("SW_GEMM_STAGGER", 1);
        a.stagger = stagger;
        const CUtensorMap& ta = tmap_cached(p.W, p.w_rows, p.K, BM);
        const CUtensorMap& tb = tmap_cached(p.X, p.x_rows, p.K, bn);
        switch (p.mode) {
            case EPI_STORE: dispatch_bn<true, EPI_STORE>(bn, ta, tb, a, st); break;
            case EPI_RESID: dispatch_bn<true, EPI_RESID>(bn, ta, tb, a, st); break;
            case EPI_SWIGLU: dispatch_bn<true, EPI_SWIGLU>(bn, ta, tb, a, st); break;
            case EPI_ARGMAX: dispatch_bn<true, EPI_ARGMAX>(bn, ta, tb, a, st); break;
            case EPI_STORE_F32: dispatch_bn<true, EPI_STORE_F32>(bn, ta, tb, a, st); break;
            case EPI_QKV_ROPE: dispatch_bn<true, EPI_QKV_ROPE>(bn, ta, tb, a, st); break;
            default: throw_cuda("gemm: bad epilogue", cudaErrorInvalidValue, __FILE__, __LINE__);
        }
    } else {
        const int bn = 256;
        if (p.features % bn != 0)
            throw_cuda("gemm: feature count must be a multiple of 256", cudaErrorInvalidValue, __FILE__, __LINE__);
        a.M = p.tokens;
        a.N = p.features;
        const CUtensorMap& ta = tmap_cached(p.X, p.x_rows, p.K, BM);
        const CUtensorMap& tb = tmap_cached(p.W, p.w_rows, p.K, bn);
        switch (p.mode) {
            case EPI_STORE: dispatch_bn<false, EPI_STORE>(bn, ta, tb, a, st); break;
            case EPI_RESID: dispatch_bn<false, EPI_RESID>(bn, ta, tb, a, st); break;
            case EPI_SWIGLU: dispatch_bn<false, EPI_SWIGLU>(bn, ta, tb, a, st); break;
            case EPI_STORE_F32: dispatch_bn<false, EPI_STORE_F32>(bn, ta, tb, a, st); break;
            default: throw_cuda("gemm: bad epilogue for normal mode", cudaErrorInvalidValue, __FILE__, __LINE__);
        }
    }
}

}  // namespace sw

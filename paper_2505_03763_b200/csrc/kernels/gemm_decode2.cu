// Decode projection GEMM for sm_100a for projections wider than the GPU (used for
// the Llama-8B gate/up at > 128 rows): swap-AB tcgen05 over a persistent grid of
// one CTA per SM, every SM streaming the same weight bytes.
//
//   Y[t, f] = sum_k X[t, k] W[f, k]   W: weights bf16 [F, K] (UMMA M = 128 rows)
//                                     X: decode rows bf16 [BN, K] (UMMA N = BN)
//
// The 8B gate/up has 224 feature tiles of 128 rows: 1.51 waves on 148 SMs, so
// the cluster split-K form (gemm_decode.cu) leaves 76 SMs with two tiles and 72
// with one, and at 256 rows the doubled SMs' MMAs set the time.  Here each of
// the P CTAs takes w = T / P whole tiles plus an equal stream-K share of the
// remaining T - w*P tiles (their (tile, 64-wide K-block) units numbered
// tile-major, CTA c taking units [c*R/P, (c+1)*R/P)).  A CTA's work is a list of
// pieces (tile, K-blocks [kb0, kb1)), its stream-K pieces FIRST; each piece
// accumulates into one of two TMEM accumulators (the epilogue of piece i
// overlaps the MMAs of piece i+1):
//   * a cut tile: every piece parks its fp32 partial token-major in an L2
//     scratch and counts itself in; after its last cut piece each of the np
//     CTAs waits for the count and reduces its 1/np of the tile's tokens -- the
//     np partials added in K order (deterministic: the pieces depend on the
//     weight shape and P only, never on the batch) -- and emits them, while the
//     MMA warp runs the whole tiles;
//   * a whole tile: TMEM (thread = feature) -> smem token-major -> one warp per
//     token runs the fused epilogue (emit_tok: residual + RMSNorm sums, SwiGLU,
//     RoPE + paged KV).  The last one is the only work left after the last MMA:
//     warps 4-7 emit its tokens 0-127 and warps 0-3 (idle by then) tokens
//     128-255, each set transposing through a drained ring.
// Warps: 0 weight TMA (never waits for the predecessor: weights are constant,
// so the ring fills under programmatic dependent launch), 1 activation TMA
// (after griddepcontrol.wait), 2 MMA issuer (UMMA N trimmed to the live rows),
// 3 spare, 4-7 epilogue.  Weight and activation rings are separate: at b = 256
// an activation k-block is twice a weight k-block, and only the weights come
// from HBM.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_decode_epi.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_sm100.cuh"

namespace sw {

namespace {

using namespace dec_epi;

__device__ unsigned long long g_dsk_trace[256][8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DSK_STAMP(i) \
    do {                                              \
        if (pl.trace && c < 256) g_dsk_trace[c][i] = gtimer(); \
    } while (0)

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr int kTs = BM + 4;  // token-major transpose row stride (floats): conflict-free, 16 B aligned

template <int BN>
struct SkCfg {
    static constexpr int kW = BM * BK * 2;  // one weight k-block: 16 KB
    static constexpr int kX = BN * BK * 2;  // one activation k-block
    static constexpr int kXtRaw = 2 * 32 * kTs * 4;  // two 32-token transpose buffers
    static constexpr int kTok = 256 * 16;            // tok_inv, tok_pos, tok_kv
    static constexpr int kBudget = 224 * 1024;
    static constexpr int NX = BN >= 128 ? 3 : 4;  // activations from L2: ~1 us of k-blocks in flight
    // The only whole tile of a CTA is its last piece (the host keeps tiles < 2 x CTAs), whose epilogue
    // runs after the last MMA: the transpose buffers alias the drained activation ring when it is large
    // enough, and the weight ring takes the space (BN = 256: 7 weight stages instead of 5).
    static constexpr bool kXtAlias = NX * kX >= kXtRaw;
    static constexpr int kXt = kXtAlias ? 0 : kXtRaw;
    static constexpr int NWraw = (kBudget - 1024 - 512 - kXt - kTok - NX * kX) / kW;
    static constexpr int NW = NWraw > 8 ? 8 : NWraw;
    static_assert(NW >= 4, "weight ring too shallow");
    static constexpr int kOffX = NW * kW;
    static constexpr int kOffXt = kXtAlias ? kOffX : kOffX + NX * kX;
    static constexpr int kOffTok = kOffX + NX * kX + kXt;
    static constexpr int kOffBar = kOffTok + kTok;
    static constexpr int kSmem = 1024 + kOffBar + 512;
    static constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
};

// Work plan (identical in every role).  The T feature tiles of the projection
// are dealt as w = T / P whole tiles per CTA (data parallel: no reduction) plus
// a remainder of rem = T - w*P tiles whose (tile, K-block) units are numbered
// tile-major, R = rem * nk of them, and cut into P equal stream-K ranges: CTA c
// takes units [c*R/P, (c+1)*R/P) of the remainder, then its w whole tiles.
// Every SM streams the same number of weight bytes; only the remainder tiles
// are reduced, and since every CTA runs its stream-K range FIRST their partials
// are in L2 early and their reductions overlap the MMAs of the whole tiles.
struct SkPlan {
    int U, P, nk;  // U = R: stream-K units of the remainder tiles
    int T, w;      // feature tiles, whole tiles per CTA
    int trace;     // SW_DSK_TRACE=1: per-CTA globaltimer phase stamps (tools/dsk_trace.py)
    __device__ __forceinline__ int t0() const { return w * P; }  // first remainder tile
    __device__ __forceinline__ int start(int c) const { return static_cast<int>(static_cast<long long>(c) * U / P); }
    // first CTA whose range holds unit x
    __device__ __forceinline__ int cta_of(int x) const {
        const int c = static_cast<int>((static_cast<long long>(x + 1) * P + U - 1) / U) - 1;
        return c < P - 1 ? c : P - 1;
    }
};

struct Piece {
    int tile, kb0, kb1, np, idx;  // idx: this CTA's position among the tile's np pieces
};
__device__ __forceinline__ Piece piece_at(const SkPlan& pl, int c, int u) {
    Piece p;
    const int rt = u / pl.nk;  // remainder tile
    p.tile = pl.t0() + rt;
    p.kb0 = u - rt * pl.nk;
    const int u1 = pl.start(c + 1);
    p.kb1 = min(pl.nk, p.kb0 + (u1 - u));
    const int cf = pl.cta_of(rt * pl.nk), cl = pl.cta_of(rt * pl.nk + pl.nk - 1);
    p.np = cl - cf + 1;
    p.idx = c - cf;
    return p;
}
// partial slot of CTA c for (remainder) tile t: 0 if t is the tile its range starts in, else 1
__device__ __forceinline__ float* part_ptr(float* ws, const SkPlan& pl, int c, int t, int bn) {
    const int slot = pl.t0() + pl.start(c) / pl.nk == t ? 0 : 1;
    return ws + (static_cast<size_t>(c) * 2 + slot) * bn * BM;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// The pieces of CTA c in processing order: its stream-K pieces of the remainder
// tiles (a range shorter than a tile touches at most two, both cut), then its
// whole tiles.
constexpr int kMaxPieces = 8;
__device__ __forceinline__ int piece_list(const SkPlan& pl, int c, Piece (&out)[kMaxPieces]) {
    int n = 0;
    for (int u = pl.start(c), u1 = pl.start(c + 1); u < u1 && n < kMaxPieces; ++n) {
        out[n] = piece_at(pl, c, u);
        u += out[n].kb1 - out[n].kb0;
    }
    for (int j = 0; j < pl.w && n < kMaxPieces; ++j, ++n) out[n] = Piece{c * pl.w + j, 0, pl.nk, 1, 0};
    return n;
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_dsk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args,
                    SkPlan pl) {
    using C = SkCfg<BN>;
    constexpr int NW = C::NW, NX = C::NX;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sW = smem;
    uint8_t* sX = smem + C::kOffX;
    float* xt = reinterpret_cast<float*>(smem + C::kOffXt);
    float* tok_inv = reinterpret_cast<float*>(smem + C::kOffTok);
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);
    uint64_t* w_full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* w_empty = w_full + NW;
    uint64_t* x_full = w_empty + NW;
    uint64_t* x_empty = x_full + NX;
    uint64_t* acc_full = x_empty + NX;   // [2]
    uint64_t* acc_empty = acc_full + 2;  // [2] (128 epilogue arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    griddep_launch_dependents();  // the successor may launch once every CTA of this grid is resident
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = static_cast<int>(blockIdx.x);
    if (threadIdx.x == 0) DSK_STAMP(0);
    Piece pcs[kMaxPieces];
    const int npcs = piece_list(pl, c, pcs);
    // Split tail: the last piece is a whole tile (its epilogue is the only work left after the last MMA),
    // so warps 0-3 -- idle by then -- emit its tokens [128, n) while warps 4-7 emit [0, 128).
    const bool split_tail = BN > 128 && npcs > 0 && pcs[npcs - 1].np == 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NW; ++s) {
            mbar_init(&w_full[s], 1);
            mbar_init(&w_empty[s], 1);
        }
        for (int s = 0; s < NX; ++s) {
            mbar_init(&x_full[s], 1);
            mbar_init(&x_empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 128);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ weight producer
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();  // read once per step
            int i = 0;
            for (int q = 0; q < npcs; ++q) {
                const Piece& p = pcs[q];
                for (int kb = p.kb0; kb < p.kb1; ++kb, ++i) {
                    const int s = i % NW;
                    if (i >= NW) mbar_wait(&w_empty[s], ((i / NW) - 1) & 1);
                    mbar_expect_tx(&w_full[s], C::kW);
                    tma_load_2d(sW + s * C::kW, &tmA, &w_full[s], kb * BK, p.tile * BM, pol);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ activation producer
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_last();  // re-read by every tile
            griddep_wait();  // activations come from the predecessor
            int i = 0;
            for (int q = 0; q < npcs; ++q) {
                const Piece& p = pcs[q];
                for (int kb = p.kb0; kb < p.kb1; ++kb, ++i) {
                    const int s = i % NX;
                    if (i >= NX) mbar_wait(&x_empty[s], ((i / NX) - 1) & 1);
                    mbar_expect_tx(&x_full[s], C::kX);
                    tma_load_2d(sX + s * C::kX, &tmB, &x_full[s], kb * BK, 0, pol);
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ------------------------------------------------------------ MMA issuer (+ TMEM owner)
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
        tc_fence_before();
        asm volatile("bar.arrive 2, 160;" ::: "memory");  // publish the TMEM address to the epilogue warps
        tc_fence_after();
        const uint32_t tmem = *tmem_slot;
        if (lane == 0) {
            // UMMA N trimmed to the live rows (multiple of 16): a bucket of BN rows computes only the
            // columns in use; each output column's K order is unchanged (results bit-identical)
            // (the count is loaded now and used after the first stage lands, so its latency hides there)
            griddep_wait();  // the live row count comes from the predecessor
            const int live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
            uint32_t idesc = 0;
            int i = 0;
            for (int q = 0; q < npcs; ++q) {
                const Piece& p = pcs[q];
                const int ab = q & 1;
                if (q >= 2) mbar_wait(&acc_empty[ab], ((q >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t acc = tmem + ab * BN;
                for (int kb = p.kb0; kb < p.kb1; ++kb, ++i) {
                    const int sw = i % NW, sx = i % NX;
                    mbar_wait(&w_full[sw], (i / NW) & 1);
                    mbar_wait(&x_full[sx], (i / NX) & 1);
                    if (i == 0) idesc = umma_idesc_bf16(BM, min(BN, max(16, (live + 15) & ~15)));
                    tc_fence_after();
                    if (i == 0) DSK_STAMP(1);
                    const uint32_t a0 = smem_addr(sW + sw * C::kW);
                    const uint32_t b0 = smem_addr(sX + sx * C::kX);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        umma_bf16(acc, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                                  (kb > p.kb0 || k > 0) ? 1u : 0u);
                    umma_commit(&w_empty[sw]);
                    umma_commit(&x_empty[sx]);
                }
                umma_commit(&acc_full[ab]);
            }
            DSK_STAMP(2);
        }
        __syncwarp();
    } else if (warp >= kEpiWarp0) {
        // ------------------------------------------------------------ epilogue
        asm volatile("bar.sync 2, 160;" ::: "memory");
        tc_fence_after();
        const uint32_t tmem = *tmem_slot;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;  // weight row in the tile (TMEM lane)
        const int ew = warp - kEpiWarp0;
        const int e = threadIdx.x - kEpiWarp0 * 32;
        griddep_wait();
        const int n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        fill_tok_tables<MODE>(args, n_live, e, 128, tok_inv, tok_pos, tok_kv);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (split_tail) asm volatile("bar.arrive 4, 256;" ::: "memory");  // token tables, TMEM base -> warps 0-3
        const uint32_t tb = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        int buf = 0, nred = 0;
        unsigned* done = args.counters + pl.T;
        for (int q = 0; q < npcs; ++q) {
            const Piece& p = pcs[q];
            const int ab = q & 1;
            mbar_wait(&acc_full[ab], (q >> 1) & 1);
            tc_fence_after();
            uint32_t r[32];
            const TokCtx tc{&args, tok_inv, tok_pos, tok_kv, p.tile * BM};
            if (p.np == 1) {
                // whole tile: TMEM (thread = feature) -> smem token-major -> one warp per token; the last
                // whole tile's tokens >= 128 go to warps 0-3 (split tail)
                const int c_end = split_tail && q + 1 == npcs ? min(n_live, 128) : n_live;
                for (int c0 = 0; c0 < c_end; c0 += 32, buf ^= 1) {
                    tmem_ld32(tb + ab * BN + c0, r);
                    tmem_ld_wait();
                    float* T = xt + buf * 32 * kTs;
#pragma unroll
                    for (int j = 0; j < 32; ++j) T[j * kTs + row] = __uint_as_float(r[j]);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    const int cnt = min(32, c_end - c0);
                    for (int j = ew; j < cnt; j += 4)
                        emit_tok<MODE>(tc, c0 + j, lane, *reinterpret_cast<const float4*>(T + j * kTs + 4 * lane),
                                       pre_tok<MODE>(tc, c0 + j, lane));
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[ab]);
                continue;
            }
            // cut tile: park this piece's partial token-major (a warp stores 128 contiguous bytes per token)
            float* part = part_ptr(args.ws, pl, c, p.tile, BN);
            for (int c0 = 0; c0 < n_live; c0 += 32) {
                tmem_ld32(tb + ab * BN + c0, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (c0 + j < n_live) __stcg(part + static_cast<size_t>(c0 + j) * BM + row, __uint_as_float(r[j]));
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[ab]);
            asm volatile("bar.sync 1, 128;" ::: "memory");  // all 128 rows stored
            if (e == 0) {
                __threadfence();
                atomicAdd(&args.counters[p.tile], 1u);
            }
            // after the last cut piece: reduce this CTA's token slices of every cut tile (the MMA warp
            // meanwhile runs the whole tiles)
            if (q + 1 < npcs && pcs[q + 1].np > 1) continue;
            for (int r2 = 0; r2 <= q; ++r2) {
                const Piece& s = pcs[r2];
                if (e == 0) {
                    while (ld_acquire_gpu(&args.counters[s.tile]) < static_cast<unsigned>(s.np)) __nanosleep(32);
                    DSK_STAMP(4 + 2 * nred);
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const int cf = c - s.idx;
                const int t0 = s.idx * n_live / s.np, t1 = (s.idx + 1) * n_live / s.np;
                const TokCtx sc{&args, tok_inv, tok_pos, tok_kv, s.tile * BM};
                // memory-level parallelism: a warp reduces kTR tokens at a time, kKB partials of each in
                // flight together (16 float4 loads per lane)
                constexpr int kEw = 4, kTR = 8, kKB = 2;
                for (int tq = t0 + ew; tq < t1; tq += kEw * kTR) {
                    float4 v[kTR];
                    TokPre pre[kTR];
#pragma unroll
                    for (int z = 0; z < kTR; ++z) {
                        v[z] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (tq + z * kEw < t1) pre[z] = pre_tok<MODE>(sc, tq + z * kEw, lane);
                    }
                    for (int k0 = 0; k0 < s.np; k0 += kKB) {
                        float4 in[kTR][kKB];
                        const float4* src[kKB];
#pragma unroll
                        for (int k = 0; k < kKB; ++k)
                            src[k] = reinterpret_cast<const float4*>(
                                         part_ptr(args.ws, pl, cf + min(k0 + k, s.np - 1), s.tile, BN)) + lane;
#pragma unroll
                        for (int z = 0; z < kTR; ++z)
#pragma unroll
                            for (int k = 0; k < kKB; ++k)
                                if (tq + z * kEw < t1 && k0 + k < s.np)
                                    in[z][k] = __ldcg(src[k] + static_cast<size_t>(tq + z * kEw) * (BM / 4));
#pragma unroll
                        for (int z = 0; z < kTR; ++z)
#pragma unroll
                            for (int k = 0; k < kKB; ++k)
                                if (k0 + k < s.np) {  // K order: deterministic
                                    v[z].x += in[z][k].x;
                                    v[z].y += in[z][k].y;
                                    v[z].z += in[z][k].z;
                                    v[z].w += in[z][k].w;
                                }
                    }
#pragma unroll
                    for (int z = 0; z < kTR; ++z)
                        if (tq + z * kEw < t1) emit_tok<MODE>(sc, tq + z * kEw, lane, v[z], pre[z]);
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (e == 0) {
                    // the tile's last reducer re-arms both counters for the next launch (every other
                    // reducer of the tile has passed its wait by now)
                    if (atomicAdd(&done[s.tile], 1u) == static_cast<unsigned>(s.np - 1)) {
                        args.counters[s.tile] = 0u;
                        done[s.tile] = 0u;
                    }
                    DSK_STAMP(5 + 2 * nred);
                }
                ++nred;
            }
        }
    }
    if (split_tail && warp < kEpiWarp0) {
        // ------------------------------------------------------------ split tail (warps 0-3)
        asm volatile("bar.sync 4, 256;" ::: "memory");  // token tables filled, TMEM base published
        griddep_wait();
        const int n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        if (n_live > 128) {
            const int q = npcs - 1, ab = q & 1;
            mbar_wait(&acc_full[ab], (q >> 1) & 1);  // the last MMA retired: the weight ring is free
            tc_fence_after();
            const uint32_t tb = *tmem_slot + (static_cast<uint32_t>(warp * 32) << 16) + ab * BN;
            const int row = warp * 32 + lane;
            float* xb = reinterpret_cast<float*>(sW);  // two 32-token transpose buffers in the drained ring
            const TokCtx tc{&args, tok_inv, tok_pos, tok_kv, pcs[q].tile * BM};
            int buf = 0;
            for (int c0 = 128; c0 < n_live; c0 += 32, buf ^= 1) {
                uint32_t r[32];
                tmem_ld32(tb + c0, r);
                tmem_ld_wait();
                float* T = xb + buf * 32 * kTs;
#pragma unroll
                for (int j = 0; j < 32; ++j) T[j * kTs + row] = __uint_as_float(r[j]);
                asm volatile("bar.sync 3, 128;" ::: "memory");
                const int cnt = min(32, n_live - c0);
                for (int j = warp; j < cnt; j += 4)
                    emit_tok<MODE>(tc, c0 + j, lane, *reinterpret_cast<const float4*>(T + j * kTs + 4 * lane),
                                   pre_tok<MODE>(tc, c0 + j, lane));
            }
            tc_fence_before();
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) DSK_STAMP(7);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(*tmem_slot, C::kTmemCols);
    }
}

template <int BN, int MODE>
void launch_dsk(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, const SkPlan& pl, cudaStream_t st) {
    using C = SkCfg<BN>;
    static bool configured = false;
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_dsk_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        configured = true;
    }
    launch_k(gemm_dsk_kernel<BN, MODE>, dim3(pl.P), dim3(kThreads), C::kSmem, st, a, b, args, pl);
}

template <int BN>
void dispatch_dsk(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, const SkPlan& pl,
                  cudaStream_t st) {
    switch (args.mode) {
        case EPI_STORE: launch_dsk<BN, EPI_STORE>(a, b, args, pl, st); break;
        case EPI_RESID: launch_dsk<BN, EPI_RESID>(a, b, args, pl, st); break;
        case EPI_SWIGLU: launch_dsk<BN, EPI_SWIGLU>(a, b, args, pl, st); break;
        case EPI_STORE_F32: launch_dsk<BN, EPI_STORE_F32>(a, b, args, pl, st); break;
        case EPI_QKV_ROPE: launch_dsk<BN, EPI_QKV_ROPE>(a, b, args, pl, st); break;
        default: throw_cuda("gemm_decode_sk: unsupported epilogue", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace

// Scratch of the stream-K decode GEMM on P CTAs: two partial tiles per CTA, and
// two counters (arrivals, reducers) per feature tile.
size_t gemm_decode_sk_ws_floats(int P, int bn) { return static_cast<size_t>(P) * 2 * bn * BM; }

void gemm_decode_sk_run(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int bn, int tiles, int P,
                        cudaStream_t st) {
    static const int trace = [] {
        const char* v = std::getenv("SW_DSK_TRACE");
        return v && *v ? std::atoi(v) : 0;
    }();
    const int nk = args.K / BK, w = tiles / P;
    SkPlan pl{(tiles - w * P) * nk, P, nk, tiles, w, trace};
    switch (bn) {
        case 32: dispatch_dsk<32>(a, b, args, pl, st); break;
        case 64: dispatch_dsk<64>(a, b, args, pl, st); break;
        case 128: dispatch_dsk<128>(a, b, args, pl, st); break;
        case 256: dispatch_dsk<256>(a, b, args, pl, st); break;
        default: throw_cuda("gemm_decode_sk: unsupported BN", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace sw

// debug: the per-CTA phase stamps of the last traced launch (SW_DSK_TRACE=1)
extern "C" int sw_dbg_dsk_trace(unsigned long long* host, int n) {
    if (n > 256 * 8) n = 256 * 8;
    return cudaMemcpyFromSymbol(host, sw::g_dsk_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}

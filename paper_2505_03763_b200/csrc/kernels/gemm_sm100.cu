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
// Persistent kernel, one CTA per SM, 8 warps:
//   warp 0    barrier init, tensor-map prefetch
//   warp 1    TMEM allocator + MMA issuer (one lane): 4 x tcgen05.mma
//             (128 x BN x 16) per 64-wide K-block into one of two TMEM
//             accumulators; tcgen05.commit frees the smem stage / publishes
//             the accumulator
//   warps 2-3 TMA producers, interleaved over K-blocks (one issuing thread
//             completes only ~1 bulk copy per ~600 cycles, tools/tma_bench2.cu)
//   warps 4-7 epilogue: tcgen05.ld 32x32b.x32 (warp%4 picks its TMEM lane
//             quarter) -> fused epilogue -> global, overlapping the MMAs of
//             the next tile through the double-buffered accumulator.
// Work split:
//   prefill  whole 128 x BN tiles, round robin over the CTAs;
//   decode   stream-K: the (tile, K-block) iterations are divided evenly over
//            the CTAs, so every SM streams the same number of weight bytes
//            whatever the tile count; a tile split across CTAs is reduced by
//            the last CTA to finish it, adding the partials in CTA order
//            (deterministic, batch independent).
// Epilogues: STORE (bf16), STORE_F32, RESID (fp32 residual +=), SWIGLU over
// [gate 64 | up 64] feature blocks, ARGMAX (packed 64-bit atomicMax per token:
// LM head + greedy sampling in one pass), QKV_ROPE (decode: RMSNorm scale,
// RoPE, q to a buffer and k/v straight into the paged KV cache).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_sm100.cuh"

namespace sw {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kProducers = 2;
constexpr int kThreads = 256;  // 8 warps
constexpr int kEpiBase = 128;  // first epilogue thread (warp 4)
constexpr int kMaxContrib = 8;  // stream-K: CTAs contributing to one tile (host enforces)

// LEAN (prefill, BN = 128): ~105 KB of smem and 256 TMEM columns, so a decode
// CTA (<= ~104 KB, <= 128 columns) fits on the same SM -- the co-resident
// prefill the split executor launches while decode work exists.
template <int BN, bool SWAP, bool PAIR = false, bool LEANP = false>
struct GemmCfg {
    // lean: ~100 KB of smem (and, for pairs, one 256-column accumulator) so a decode CTA fits beside
    static constexpr bool kLean = (!SWAP && BN == 128) || LEANP;
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = (PAIR ? BN / 2 : BN) * BK * 2;  // PAIR: this CTA's half of the N tile
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kBudget = kLean ? 96 * 1024 : 192 * 1024;
    static constexpr int kStagesRaw = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
    static constexpr int kStages = kLean ? kStagesRaw : (kStagesRaw & ~1);
    static_assert(kStages >= (kLean ? 3 : 4), "stage ring too shallow");
    static constexpr int kAccs = LEANP ? 1 : 2;  // TMEM accumulators (double-buffered unless lean pair)
    static constexpr int kTmemCols = kAccs * BN < 64 ? 64 : kAccs * BN;
    static constexpr int kXchgBytes = SWAP ? 128 * 33 * 4 : 0;
    static constexpr int kTokBytes = 256 * 24;  // tok_inv, tok_pos, tok_kv, best
    static constexpr int kBarBytes = 512;
    static constexpr int kSmem = 1024 + kStages * kStageBytes + kXchgBytes + kTokBytes + kBarBytes;
};

// Static work schedule shared by every role of a CTA.
struct Sched {
    int tiles_n, tiles, nk, C, c;
    int tiles_m, gm;  // grouped raster: token tiles per group (normal mode)
    bool stream_k;
    long long I;  // stream-K: total (tile, K-block) iterations
    __device__ long long beg(int cc) const { return static_cast<long long>(cc) * I / C; }
    // Tile t -> (token tile, feature tile).  Grouped raster: tiles walk a group of gm token tiles
    // token-fastest, then the next feature panel, so the CTAs running at one time share a few weight
    // panels and the group's activation rows stay in L2 -- each weight panel is read from HBM once per
    // group instead of once per token tile (8B gate/up at 4096 tokens: 16 -> 1 pass over 235 MB).
    __device__ void coords(int t, int& mt, int& nt) const {
        if (gm <= 1) {
            mt = t / tiles_n;
            nt = t % tiles_n;
            return;
        }
        const int span = gm * tiles_n;
        const int grp = t / span, r = t - grp * span;
        const int rows = min(gm, tiles_m - grp * gm);
        mt = grp * gm + r % rows;
        nt = r / rows;
    }
    __device__ int owner(long long u) const {  // CTA whose range holds iteration u
        int cc = static_cast<int>((u * C) / I);
        while (cc + 1 < C && beg(cc + 1) <= u) ++cc;
        while (cc > 0 && beg(cc) > u) --cc;
        return cc;
    }
};

struct Seg {
    int tile, lo, hi;
};

struct SegIter {
    long long u, end;
    int t;
    __device__ void init(const Sched& s) {
        if (s.stream_k) {
            u = s.beg(s.c);
            end = s.beg(s.c + 1);
        } else {
            t = s.c;
        }
    }
    __device__ bool next(const Sched& s, Seg& g) {
        if (s.stream_k) {
            if (u >= end) return false;
            g.tile = static_cast<int>(u / s.nk);
            g.lo = static_cast<int>(u - static_cast<long long>(g.tile) * s.nk);
            const long long stop = min(end, static_cast<long long>(g.tile + 1) * s.nk);
            g.hi = static_cast<int>(stop - static_cast<long long>(g.tile) * s.nk);
            u = stop;
            return true;
        }
        if (t >= s.tiles) return false;
        g.tile = t;
        g.lo = 0;
        g.hi = s.nk;
        t += s.C;
        return true;
    }
};

// PAIR (prefill, BN = 256): a CTA pair (cluster of 2) computes 256 x 256 tiles
// with tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 token rows
// of A and its 128 feature rows of B (32 KB per stage instead of 48 KB for the
// same FLOPs), both CTAs' TMA loads complete on the leader's full barrier, the
// leader issues the MMAs and its commits arrive on both CTAs' barriers, and each
// CTA's epilogue drains its own 128 accumulator rows.
template <int BN, int MODE, bool SWAP, bool PAIR = false, bool LEANP = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    using C = GemmCfg<BN, SWAP, PAIR, LEANP>;
    static_assert(!LEANP || PAIR, "lean accumulators: pair kernel only");
    static_assert(!PAIR || (!SWAP && BN == 256), "CTA pairs: prefill 256-wide tiles only");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kABytes;
    float* xchg = reinterpret_cast<float*>(sB + C::kStages * C::kBBytes);                // [128][33]
    float* tok_inv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xchg) + C::kXchgBytes);  // [256]
    int* tok_pos = reinterpret_cast<int*>(tok_inv + 256);                                // [256]
    long long* tok_kv = reinterpret_cast<long long*>(tok_pos + 256);                     // [256]
    unsigned long long* best = reinterpret_cast<unsigned long long*>(tok_kv + 256);     // [256] ARGMAX
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tok_inv) + C::kTokBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* acc_full = empty + C::kStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    uint32_t* last_flag = tmem_slot + 1;

    griddep_launch_dependents();  // let the next kernel of the step start its prologue
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    uint32_t rank = 0;  // PAIR: rank in the CTA pair (0 = leader)
    if constexpr (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    constexpr int BMe = PAIR ? 2 * BM : BM;  // token rows per tile
    Sched sc;
    sc.tiles_n = args.N / BN;
    sc.tiles_m = cdiv(args.M, BMe);
    sc.tiles = sc.tiles_m * sc.tiles_n;
    // group: as many token tiles as keep ~40 MB of activation rows (BMe x K bf16 each) in L2
    sc.gm = SWAP ? 1 : max(1, min(16, static_cast<int>((40ll << 20) / (static_cast<long long>(BMe) * args.K * 2))));
    sc.nk = args.K / BK;
    sc.C = PAIR ? gridDim.x / 2 : gridDim.x;
    sc.c = PAIR ? blockIdx.x / 2 : blockIdx.x;
    sc.stream_k = args.stream_k != 0;
    sc.I = static_cast<long long>(sc.tiles) * sc.nk;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], PAIR ? 8 : 4);  // one arrive per epilogue warp (of both CTAs: PAIR)
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                         "r"(static_cast<uint32_t>(C::kTmemCols)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc(tmem_slot, C::kTmemCols);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR)  // both CTAs' barriers exist before any remote arrive / multicast commit
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // PAIR: the leader's copy of a barrier (its shared::cluster address)
    auto leader_bar = [&](uint64_t* b) {
        uint32_t r = smem_addr(b);
        if constexpr (PAIR) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(r), "r"(0));
        return r;
    };

    if (warp == 2 || warp == 3) {
        // ------------------------------------------------------------ producers
        if (lane == 0) {
            const int p = warp - 2;
            // decode (swap): weights stream once per launch (evict first), activations are re-read by
            // every tile (evict last).  Prefill: the weight panels are re-read by every token tile
            // too -- evict first sent them back to HBM between tiles (the gate/up GEMM read 3.4 GB
            // from HBM for 134 MB of operands)
            const uint64_t pol_w = SWAP ? l2_policy_evict_first() : l2_policy_evict_last();
            const uint64_t pol_x = l2_policy_evict_last();
            auto coord = [&](const Seg& g, int& am, int& bn0) {
                int mt, nt;
                sc.coords(g.tile, mt, nt);
                am = mt * BMe + static_cast<int>(rank) * BM;
                bn0 = nt * BN + (PAIR ? static_cast<int>(rank) * (BN / 2) : 0);
            };
            // TMA into this CTA's smem, completing on `full[s]` (PAIR: the leader's)
            auto load = [&](void* dst, const CUtensorMap* tm, int s, int x, int y, uint64_t pol) {
                if constexpr (PAIR) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_addr(dst)),
                        "l"(tm), "r"(leader_bar(&full[s])), "r"(x), "r"(y), "l"(pol)
                        : "memory");
                } else {
                    tma_load_2d(dst, tm, &full[s], x, y, pol);
                }
            };
            // the stage's expected bytes: PAIR -> both CTAs' loads, armed by the leader only
            auto arm = [&](int s) {
                if (!PAIR) mbar_expect_tx(&full[s], C::kStageBytes);
                else if (rank == 0) mbar_expect_tx(&full[s], 2 * C::kStageBytes);
            };
            // Pass 1 (PDL): the first ring fill of the constant operand -- the
            // weights -- is issued before waiting on the predecessor kernel.
            {
                SegIter it;
                it.init(sc);
                Seg g;
                int gi = 0;
                while (gi < C::kStages && it.next(sc, g)) {
                    int am, bn0;
                    coord(g, am, bn0);
                    for (int kb = g.lo; kb < g.hi && gi < C::kStages; ++kb, ++gi) {
                        if (gi % kProducers != p) continue;
                        arm(gi);
                        if (SWAP) load(sA + gi * C::kABytes, &tmA, gi, kb * BK, am, pol_w);
                        else load(sB + gi * C::kBBytes, &tmB, gi, kb * BK, bn0, pol_w);
                    }
                }
            }
            griddep_wait();
            SegIter it;
            it.init(sc);
            Seg g;
            int gi = 0;
            while (it.next(sc, g)) {
                int am, bn0;
                coord(g, am, bn0);
                for (int kb = g.lo; kb < g.hi; ++kb, ++gi) {
                    if (gi % kProducers != p) continue;
                    const int s = gi % C::kStages;
                    if (gi < C::kStages) {  // weights already in flight: the activation half
                        if (SWAP) load(sB + s * C::kBBytes, &tmB, s, kb * BK, bn0, pol_x);
                        else load(sA + s * C::kABytes, &tmA, s, kb * BK, am, pol_x);
                        continue;
                    }
                    mbar_wait(&empty[s], ((gi / C::kStages) & 1) ^ 1);
                    arm(s);
                    load(sA + s * C::kABytes, &tmA, s, kb * BK, am, SWAP ? pol_w : pol_x);
                    load(sB + s * C::kBBytes, &tmB, s, kb * BK, bn0, SWAP ? pol_x : pol_w);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BMe, BN);
            auto commit = [&](uint64_t* b) {  // PAIR: arrive on this barrier in both CTAs
                if constexpr (PAIR)
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
                        "[%0], %1;" ::"r"(smem_addr(b)),
                        "h"(static_cast<uint16_t>(3))
                        : "memory");
                else
                    umma_commit(b);
            };
            SegIter it;
            it.init(sc);
            Seg g;
            int gi = 0, si = 0;
            while (it.next(sc, g)) {
                const int a = si % C::kAccs;
                mbar_wait(&acc_empty[a], ((si / C::kAccs) & 1) ^ 1);
                tc_fence_after();
                const uint32_t acc = tmem + a * BN;
                for (int kb = g.lo; kb < g.hi; ++kb, ++gi) {
                    const int s = gi % C::kStages;
                    mbar_wait(&full[s], (gi / C::kStages) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_addr(sA + s * C::kABytes);
                    const uint32_t b0 = smem_addr(sB + s * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        if constexpr (PAIR)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(acc),
                                "l"(umma_desc_sw128(a0 + k * 32)), "l"(umma_desc_sw128(b0 + k * 32)), "r"(idesc),
                                "r"((kb > g.lo || k > 0) ? 1u : 0u));
                        else
                            umma_bf16(acc, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                                      (kb > g.lo || k > 0) ? 1u : 0u);
                    }
                    commit(&empty[s]);
                }
                commit(&acc_full[a]);
                ++si;
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        griddep_wait();  // predecessor outputs are read below
        const int quarter = warp & 3;             // TMEM lanes [32*quarter, +32)
        const int row = quarter * 32 + lane;      // accumulator row in the tile
        const int e = threadIdx.x - kEpiBase;     // 0..127
        const int n_live = args.live_tokens ? min(args.valid_tokens, *args.live_tokens) : args.valid_tokens;
        const DecodeFusion& fx = args.fx;
        if constexpr (SWAP) {
            // per-token epilogue inputs (the batch is one N tile), gathered once
            for (int t = e; t < BN && t < n_live; t += 128) {
                if (fx.ss_parts) {
                    float ss = 0.f;
                    for (int q = 0; q < fx.ss_nparts; ++q) ss += fx.ss_parts[q * kSsStride + t];
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
        }

        SwapEpi E{&args, xchg, tok_inv, tok_pos, tok_kv, row, lane, quarter, n_live};
        if constexpr (MODE == EPI_ARGMAX) {
            for (int t = e; t < 256; t += 128) best[t] = 0ull;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            E.best = best;
        }
        auto emit_swap_l = [&](int m0, int c, const float (&v)[32]) { emit_swap<MODE>(E, m0, c, v); };

        // normal mode: row = token m0 + row, columns = features n0 + [c, c + 32)
        auto emit_normal = [&](int m0, int n0, int c, const uint32_t (&r)[32]) {
            const int t = m0 + row;
            if (t >= n_live) return;
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
                // all loads first, then all stores: 8 requests in flight, not 8 round trips
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
        };

        auto release_acc = [&](int a) {
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR)  // the leader's MMA warp waits on its own copy
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     leader_bar(&acc_empty[a]))
                                 : "memory");
                else
                    mbar_arrive(&acc_empty[a]);
            }
        };

        SegIter it;
        it.init(sc);
        Seg g;
        int si = 0;
        uint32_t r[32];
        while (it.next(sc, g)) {
            const int a = si % C::kAccs;
            int mt, nt;
            sc.coords(g.tile, mt, nt);
            const int m0 = mt * BMe + static_cast<int>(rank) * BM, n0 = nt * BN;
            // prefill residual add: the residual row's first 32 columns load while the tile's MMAs
            // still run, and every later chunk's load is in flight one chunk ahead (the epilogue
            // was a chain of 8 dependent round trips per tile: wo ran at 26% tensor-pipe)
            float4 res_cur[8];
            const bool res_live = !SWAP && MODE == EPI_RESID && m0 + row < n_live;
            float4* res_row = reinterpret_cast<float4*>(static_cast<float*>(args.out) +
                                                        static_cast<size_t>(m0 + row) * args.ldo + n0);
            if constexpr (!SWAP && MODE == EPI_RESID) {
                if (res_live) {
                    // the whole BN-column residual row of this thread into L2 while the tile's MMAs run
                    // (measured: a tile earlier was slower; wo GEMM 234 -> 183 us)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(res_row), "r"(BN * 4) : "memory");
#pragma unroll
                    for (int q = 0; q < 8; ++q) res_cur[q] = __ldcg(res_row + q);
                }
            }
            mbar_wait(&acc_full[a], (si / C::kAccs) & 1);
            tc_fence_after();
            ++si;
            const uint32_t tb = tmem + a * BN + (static_cast<uint32_t>(quarter * 32) << 16);
            const bool whole = g.lo == 0 && g.hi == sc.nk;
            if constexpr (!SWAP) {
                // prefill: whole tiles only
                if constexpr (MODE == EPI_SWIGLU) {
                    for (int blk = 0; blk < BN / 128; ++blk) {
#pragma unroll
                        for (int half = 0; half < 64; half += 32) {
                            uint32_t u[32];
                            tmem_ld32(tb + blk * 128 + half, r);
                            tmem_ld32(tb + blk * 128 + 64 + half, u);
                            tmem_ld_wait();
                            if (blk == BN / 128 - 1 && half == 32) release_acc(a);
                            const int t = m0 + row;
                            if (t < n_live) {
                                uint4* d4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.out) +
                                                                     static_cast<size_t>(t) * args.ldo +
                                                                     (n0 + blk * 128) / 2 + half);
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
                } else if constexpr (MODE == EPI_QKV_ROPE) {
                    // prefill QKV projection with RoPE and the paged-KV write fused (the rope_kv
                    // pass over an fp32 QKV buffer it replaces): the tile's BN columns are whole
                    // heads; this thread's row is one token.  Same formula and rounding points as
                    // rope_kv_kernel: fp32 rotate-half, one bf16 rounding.
                    const int t = m0 + row;
                    const bool live = t < n_live;
                    int pos = 0;
                    long long kv_off = 0;
                    if (live) {
                        pos = fx.pos[t];
                        const int page = fx.page_table[static_cast<long long>(fx.slot[t]) * fx.max_pages +
                                                       pos / fx.page_tokens];
                        kv_off = static_cast<long long>(page) * fx.page_stride +
                                 static_cast<long long>(pos % fx.page_tokens) * fx.hd;
                    }
                    const int hd = fx.hd, half = hd >> 1;
                    const long long head_stride = static_cast<long long>(fx.page_tokens) * hd;
                    for (int col0 = 0; col0 < BN; col0 += hd) {
                        const int h = (n0 + col0) / hd;
                        // one head: hd / 32 chunks; pair i is (i, i + half) = chunk c, lane-column j
                        // with chunk c + hd / 64
                        for (int c = 0; c < hd / 64; ++c) {
                            uint32_t u[32];
                            tmem_ld32(tb + col0 + c * 32, r);
                            tmem_ld32(tb + col0 + half + c * 32, u);
                            tmem_ld_wait();
                            if (col0 + hd == BN && c == hd / 64 - 1) release_acc(a);
                            if (!live) continue;
                            uint32_t pa[16], pb[16];
                            if (h < fx.H + fx.Hkv) {
                                const float2* cs = fx.rope_cs + static_cast<long long>(pos) * half + c * 32;
#pragma unroll
                                for (int j = 0; j < 32; j += 2) {
                                    const float2 c0 = cs[j], c1 = cs[j + 1];
                                    const float a0 = __uint_as_float(r[j]), b0 = __uint_as_float(u[j]);
                                    const float a1 = __uint_as_float(r[j + 1]), b1 = __uint_as_float(u[j + 1]);
                                    pa[j / 2] = pack_h2(a0 * c0.x - b0 * c0.y, a1 * c1.x - b1 * c1.y);
                                    pb[j / 2] = pack_h2(b0 * c0.x + a0 * c0.y, b1 * c1.x + a1 * c1.y);
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; j += 2) {
                                    pa[j / 2] = pack_h2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
                                    pb[j / 2] = pack_h2(__uint_as_float(u[j]), __uint_as_float(u[j + 1]));
                                }
                            }
                            kv_t* dst;
                            if (h < fx.H) {
                                dst = fx.q_out + static_cast<long long>(t) * fx.H * hd + static_cast<long long>(h) * hd;
                            } else if (h < fx.H + fx.Hkv) {
                                dst = fx.kv_layer + kv_off + (h - fx.H) * head_stride;
                            } else {
                                dst = fx.kv_layer + kv_off + fx.page_stride / 2 + (h - fx.H - fx.Hkv) * head_stride;
                            }
                            uint4* da = reinterpret_cast<uint4*>(dst + c * 32);
                            uint4* db = reinterpret_cast<uint4*>(dst + half + c * 32);
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                da[v] = make_uint4(pa[4 * v], pa[4 * v + 1], pa[4 * v + 2], pa[4 * v + 3]);
                                db[v] = make_uint4(pb[4 * v], pb[4 * v + 1], pb[4 * v + 2], pb[4 * v + 3]);
                            }
                        }
                    }
                } else if constexpr (MODE == EPI_RESID) {
                    for (int c = 0; c < BN; c += 32) {
                        float4 res_nxt[8];
                        if (res_live && c + 32 < BN) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) res_nxt[q] = __ldcg(res_row + (c + 32) / 4 + q);
                        }
                        tmem_ld32(tb + c, r);
                        tmem_ld_wait();
                        if (c == BN - 32) release_acc(a);
                        if (res_live) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                float4 v = res_cur[q];
                                v.x += __uint_as_float(r[4 * q + 0]);
                                v.y += __uint_as_float(r[4 * q + 1]);
                                v.z += __uint_as_float(r[4 * q + 2]);
                                v.w += __uint_as_float(r[4 * q + 3]);
                                res_row[c / 4 + q] = v;
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) res_cur[q] = res_nxt[q];
                    }
                } else {
                    for (int c = 0; c < BN; c += 32) {
                        tmem_ld32(tb + c, r);
                        tmem_ld_wait();
                        if (c == BN - 32) release_acc(a);
                        emit_normal(m0, n0, c, r);
                    }
                }
            } else if (whole) {
                for (int c = 0; c < BN; c += 32) {
                    tmem_ld32(tb + c, r);
                    tmem_ld_wait();
                    if (c == BN - 32) release_acc(a);
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                    emit_swap_l(m0, c, v);
                }
            } else {
                // stream-K partial tile: park it, the last contributor reduces
                const long long t0 = static_cast<long long>(g.tile) * sc.nk;
                const int c_first = sc.owner(t0), c_last = sc.owner(t0 + sc.nk - 1);
                const int slot = sc.beg(sc.c) >= t0 ? 0 : 1;  // the CTA's first or last segment
                // partial layout [BN/8][128 rows][8]: a thread's 8 columns are 32 contiguous bytes
                float* part = args.ws + (static_cast<size_t>(sc.c) * 2 + slot) * BN * 128;
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
                release_acc(a);
                __threadfence();
                asm volatile("bar.sync 2, 128;" ::: "memory");
                if (e == 0) {
                    const unsigned prev = atomicAdd(args.counters + g.tile, 1u);
                    *last_flag = prev == static_cast<unsigned>(c_last - c_first);
                }
                asm volatile("bar.sync 2, 128;" ::: "memory");
                if (*last_flag) {
                    __threadfence();
                    const int ncon = c_last - c_first + 1;
                    for (int c = 0; c < BN; c += 32) {
                        float v[32];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {  // 8 columns at a time, every contributor's load in flight
                            float4 lo[kMaxContrib], hi[kMaxContrib];
#pragma unroll
                            for (int k = 0; k < kMaxContrib; ++k) {
                                if (k < ncon) {
                                    const int cc = c_first + k;
                                    const int sl = sc.beg(cc) >= t0 ? 0 : 1;
                                    const float4* pp = reinterpret_cast<const float4*>(
                                        args.ws + (static_cast<size_t>(cc) * 2 + sl) * BN * 128 +
                                        (static_cast<size_t>(c / 8 + q) * 128 + row) * 8);
                                    lo[k] = __ldcg(pp);
                                    hi[k] = __ldcg(pp + 1);
                                }
                            }
                            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                            for (int k = 0; k < kMaxContrib; ++k) {  // contributor (CTA) order: deterministic
                                if (k < ncon) {
                                    acc[0] += lo[k].x; acc[1] += lo[k].y; acc[2] += lo[k].z; acc[3] += lo[k].w;
                                    acc[4] += hi[k].x; acc[5] += hi[k].y; acc[6] += hi[k].z; acc[7] += hi[k].w;
                                }
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) v[8 * q + j] = acc[j];
                        }
                        emit_swap_l(m0, c, v);
                    }
                    if (e == 0) args.counters[g.tile] = 0u;  // re-arm for the next launch
                }
                asm volatile("bar.sync 2, 128;" ::: "memory");  // last_flag reuse
            }
        }
        if constexpr (MODE == EPI_ARGMAX) {  // flush the CTA's per-token maxima
            asm volatile("bar.sync 1, 128;" ::: "memory");
            for (int t = e; t < BN && t < n_live; t += 128)
                if (best[t]) atomicMax(args.argmax + t, best[t]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) {  // both CTAs done: no remote arrive or multicast commit is still in flight
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (warp == 1) {
            tc_fence_after();
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                         "r"(static_cast<uint32_t>(C::kTmemCols)));
        }
    } else if (warp == 1) {
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

int env_flag(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 0;
        SW_CUDA(cudaGetDevice(&dev));
        SW_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

template <int BN, int MODE, bool SWAP>
void launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int ctas, cudaStream_t st) {
    using C = GemmCfg<BN, SWAP>;
    static bool configured = false;  // per instantiation
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, MODE, SWAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::kSmem));
        configured = true;
    }
    launch_k(gemm_tc_kernel<BN, MODE, SWAP>, dim3(ctas), dim3(kThreads), C::kSmem, st, a, b, args);
}

// CTA-pair prefill GEMM (BN = 256): clusters of 2, one pair per two SMs.
template <int MODE, bool LEANP = false>
void launch_pair(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int pairs, cudaStream_t st) {
    using C = GemmCfg<256, false, true, LEANP>;
    static bool configured = false;
    if (!configured) {
        SW_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<256, MODE, false, true, LEANP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
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
    SW_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<256, MODE, false, true, LEANP>, a, b, args));
    count_launches(1);
}

template <bool SWAP, int MODE>
void dispatch_bn(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int ctas, cudaStream_t st) {
    switch (bn) {
        case 32: launch_one<32, MODE, SWAP>(a, b, args, ctas, st); break;
        case 64: launch_one<64, MODE, SWAP>(a, b, args, ctas, st); break;
        case 128: launch_one<128, MODE, SWAP>(a, b, args, ctas, st); break;
        case 256: launch_one<256, MODE, SWAP>(a, b, args, ctas, st); break;
        default: throw_cuda("gemm: unsupported BN", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
}

}  // namespace

CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, bool fp16) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_cuda("cuTensorMapEncodeTiled", cudaErrorInvalidValue, __FILE__, __LINE__);
    return m;
}

// [rows][heads][hd] fp16 (roped q, kv_t) as a 3-D map (hd, heads, rows), box 64 x 1 x 128,
// SWIZZLE_128B: one head's 128-row x 64-column tile per load.
CUtensorMap make_tmap_heads(const void* base, uint64_t rows, uint64_t heads, uint64_t hd) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {hd, heads, rows};
    const cuuint64_t strides[2] = {hd * 2, heads * hd * 2};
    const cuuint32_t box[3] = {64, 1, 128};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_cuda("cuTensorMapEncodeTiled (3d)", cudaErrorInvalidValue, __FILE__, __LINE__);
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

int stream_sm_count(cudaStream_t st);  // engine/partition.cu

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
    a.fx = p.fx;
    a.ws = p.ws;
    a.counters = p.counters;
    const int sms = num_sms();             // device: fixes the split-K factors (numerics)
    const int grid_sms = stream_sm_count(st);  // the stream's SM partition: sizes persistent grids
    if (p.swap) {
        if (p.features % BM != 0)
            throw_cuda("gemm(swap): feature count must be a multiple of 128", cudaErrorInvalidValue, __FILE__, __LINE__);
        if (p.tokens > 256) throw_cuda("gemm(swap): at most 256 tokens", cudaErrorInvalidValue, __FILE__, __LINE__);
        const int bn = gemm_pick_bn_swap(p.tokens);
        a.M = p.features;
        a.N = bn;
        const int tiles = p.features / BM;
        static const int dec_env = env_flag("SW_GEMM_DEC", 1);
        if (dec_env && p.mode != EPI_ARGMAX && p.ws) {
            // decode projections: cluster split-K, column-distributed reduction
            // two CTAs per SM fit (<= 112 KB smem each); measured: 2 x SMs beats 1 x SMs
            // on the Llama-1B step (tools/profile_step.py)
            // more feature tiles than SMs (Llama-8B gate/up: 224 tiles): gemm_decode2.cu deals each SM
            // tiles / SMs whole tiles plus an equal stream-K share of the remainder tiles, so every SM
            // streams the same weight bytes (the cluster form below leaves 76 SMs with two tiles and 72
            // with one: at b > 128 rows the MMAs of the doubled SMs set the time).  Gates (SW_GEMM_DSK=0
            // disables): rows > SW_DSK_MINBN (128: at b <= 128 the cluster form measured faster in-step) and >= SW_DSK_MINU K-blocks of remainder per CTA.
            static const int dsk_env = env_flag("SW_GEMM_DSK", 1);
            static const int dsk_minu = std::max(1, env_flag("SW_DSK_MINU", 8));
            static const int dsk_minbn = env_flag("SW_DSK_MINBN", 128);
            if (dsk_env && tiles > grid_sms && tiles < 2 * grid_sms && bn > dsk_minbn) {
                const int P = grid_sms, nk = p.K / BK;
                const int rem = tiles % P;
                if ((rem == 0 || rem * nk / P >= dsk_minu) && gemm_decode_sk_ws_floats(P, bn) <= p.ws_floats &&
                    p.counters && 2 * tiles <= p.n_counters) {
                    a.stream_k = 0;
                    gemm_decode_sk_run(tmap_cached(p.W, p.w_rows, p.K, BM), tmap_cached(p.X, p.x_rows, p.K, bn), a, bn,
                                       tiles, P, st);
                    return;
                }
            }
            static const int dec_ctas = env_flag("SW_DEC_CTAS", 0);
            static const int s_qkv = env_flag("SW_DEC_S_QKV", 0);  // experiment: fixed split for the QKV projection
            // (the experiment knob is clamped like the rule: a portable cluster of <= 8, >= 2 K-blocks per rank)
            const int S = p.mode == EPI_QKV_ROPE && s_qkv > 0
                              ? std::max(1, std::min({s_qkv, 8, p.K / BK / 2}))
                              : gemm_decode_splits(tiles, p.K / BK, dec_ctas > 0 ? dec_ctas : 2 * sms);
            static const int dec_log = env_flag("SW_DEC_LOG", 0);
            if (dec_log) {
                static std::mutex mu;
                static std::map<std::tuple<int, int, int>, int> seen;
                std::lock_guard<std::mutex> lk(mu);
                if (seen.emplace(std::make_tuple(tiles, p.K, bn), S).second)
                    std::fprintf(stderr, "[gemm_decode] tiles=%d K=%d bn=%d mode=%d -> S=%d\n", tiles, p.K, bn, p.mode, S);
            }
            if (S == 1 || gemm_decode_ws_floats(tiles, S, bn) <= p.ws_floats) {
                a.stream_k = 0;
                static const int dec_trace = env_flag("SW_DEC_TRACE", 0);
                a.trace = dec_trace;
                gemm_decode_run(tmap_cached(p.W, p.w_rows, p.K, BM), tmap_cached(p.X, p.x_rows, p.K, bn), a, bn, S,
                                tiles, st);
                return;
            }
        }
        const long long iters = static_cast<long long>(tiles) * (p.K / BK);
        // Stream-K over every SM when there is split-K scratch; the split
        // depends on the weight shape only, never on the batch.
        // At most kMaxContrib CTAs per tile: each CTA gets >= nk/(kMaxContrib-1)
        // K-blocks (a CTA range can straddle two tiles).
        const int nk = p.K / BK;
        const long long min_iters = std::max(2, cdiv(nk, kMaxContrib - 1));
        const int sk_ctas = static_cast<int>(std::min<long long>(sms, iters / min_iters));
        static const int sk_env = [] {
            const char* v = std::getenv("SW_GEMM_SK");
            return v && *v ? std::atoi(v) : -1;
        }();
        // Measured (tools/gemm_shapes.py, profiles/r01/gemm_shapes.txt): stream-K only
        // pays for long-K projections over few tiles (Wd); shorter ones are
        // faster as whole tiles (no partial-tile fixup).
        const bool sk_shape = nk >= 96 && tiles * 2 <= sms;
        const bool sk = (sk_env > 0 || (sk_env < 0 && sk_shape)) && p.ws && p.counters && tiles <= p.n_counters &&
                        static_cast<size_t>(sms) * 2 * bn * BM <= p.ws_floats && sk_ctas > tiles;
        a.stream_k = sk ? 1 : 0;
        const int ctas = sk ? sk_ctas : std::min(grid_sms, tiles);
        const CUtensorMap& ta = tmap_cached(p.W, p.w_rows, p.K, BM);
        const CUtensorMap& tb = tmap_cached(p.X, p.x_rows, p.K, bn);
        switch (p.mode) {
            case EPI_STORE: dispatch_bn<true, EPI_STORE>(bn, ta, tb, a, ctas, st); break;
            case EPI_RESID: dispatch_bn<true, EPI_RESID>(bn, ta, tb, a, ctas, st); break;
            case EPI_SWIGLU: dispatch_bn<true, EPI_SWIGLU>(bn, ta, tb, a, ctas, st); break;
            case EPI_ARGMAX: dispatch_bn<true, EPI_ARGMAX>(bn, ta, tb, a, ctas, st); break;
            case EPI_STORE_F32: dispatch_bn<true, EPI_STORE_F32>(bn, ta, tb, a, ctas, st); break;
            case EPI_QKV_ROPE: dispatch_bn<true, EPI_QKV_ROPE>(bn, ta, tb, a, ctas, st); break;
            default: throw_cuda("gemm: bad epilogue", cudaErrorInvalidValue, __FILE__, __LINE__);
        }
    } else {
        const int bn = p.lean ? 128 : 256;
        if (p.features % bn != 0)
            throw_cuda("gemm: feature count must be a multiple of 256", cudaErrorInvalidValue, __FILE__, __LINE__);
        a.M = p.tokens;
        a.N = p.features;
        a.stream_k = 0;
        // CTA pairs (tcgen05 cta_group::2, 256 x 256 tiles): SW_GEMM_PAIR=1 (default) for 256-wide tiles
        static const int pair_env = env_flag("SW_GEMM_PAIR", 1);
        if (pair_env && (bn == 256 || p.lean) && p.yield_tiles == 0 && grid_sms >= 2) {
            const int tiles2 = cdiv(p.tokens, 2 * BM) * (p.features / 256);
            const int pairs = std::min(grid_sms / 2, tiles2);
            const CUtensorMap& ta = tmap_cached(p.X, p.x_rows, p.K, BM);
            const CUtensorMap& tb = tmap_cached(p.W, p.w_rows, p.K, 128);
            if (p.lean) {  // co-resident with decode CTAs: 3 stages, one accumulator
                switch (p.mode) {
                    case EPI_STORE: launch_pair<EPI_STORE, true>(ta, tb, a, pairs, st); return;
                    case EPI_RESID: launch_pair<EPI_RESID, true>(ta, tb, a, pairs, st); return;
                    case EPI_SWIGLU: launch_pair<EPI_SWIGLU, true>(ta, tb, a, pairs, st); return;
                    case EPI_STORE_F32: launch_pair<EPI_STORE_F32, true>(ta, tb, a, pairs, st); return;
                    case EPI_QKV_ROPE: launch_pair<EPI_QKV_ROPE, true>(ta, tb, a, pairs, st); return;
                    default: break;
                }
            }
            switch (p.mode) {
                case EPI_STORE: launch_pair<EPI_STORE>(ta, tb, a, pairs, st); return;
                case EPI_RESID: launch_pair<EPI_RESID>(ta, tb, a, pairs, st); return;
                case EPI_SWIGLU: launch_pair<EPI_SWIGLU>(ta, tb, a, pairs, st); return;
                case EPI_STORE_F32: launch_pair<EPI_STORE_F32>(ta, tb, a, pairs, st); return;
                case EPI_QKV_ROPE: launch_pair<EPI_QKV_ROPE>(ta, tb, a, pairs, st); return;
                default: break;
            }
        }
        const int tiles = cdiv(p.tokens, BM) * (p.features / bn);
        int ctas = std::min(grid_sms, tiles);
        if (p.yield_tiles > 0) ctas = std::max(ctas, cdiv(tiles, p.yield_tiles));  // round robin over more CTAs
        const CUtensorMap& ta = tmap_cached(p.X, p.x_rows, p.K, BM);
        const CUtensorMap& tb = tmap_cached(p.W, p.w_rows, p.K, bn);
        switch (p.mode) {
            case EPI_STORE: dispatch_bn<false, EPI_STORE>(bn, ta, tb, a, ctas, st); break;
            case EPI_RESID: dispatch_bn<false, EPI_RESID>(bn, ta, tb, a, ctas, st); break;
            case EPI_SWIGLU: dispatch_bn<false, EPI_SWIGLU>(bn, ta, tb, a, ctas, st); break;
            case EPI_STORE_F32: dispatch_bn<false, EPI_STORE_F32>(bn, ta, tb, a, ctas, st); break;
            case EPI_QKV_ROPE: dispatch_bn<false, EPI_QKV_ROPE>(bn, ta, tb, a, ctas, st); break;
            default: throw_cuda("gemm: bad epilogue for normal mode", cudaErrorInvalidValue, __FILE__, __LINE__);
        }
    }
}

}  // namespace sw

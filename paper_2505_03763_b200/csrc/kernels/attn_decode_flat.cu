// Decode attention, flat page-balanced and TMA-fed (sm_100a).
//
// A decode step's attention is one stream over every (row, kv head, page)
// slice of the paged KV cache.  The per-unit kernel (attention.cu, one CTA per
// (row, kv head, split)) ran in ~2 waves of short CTAs whose dependent round
// trips (page ids, Q, ring fill, drain, merge) dominated: 42% of HBM at
// Llama-1B b=64 (profiles/r01c).  Here:
//   * the grid is persistent, one CTA per SM of the stream's partition, and
//     the flat page space  W = sum_rows pages(row) * Hkv  (units (row, kv head)
//     in order, pages in order inside a unit) is cut into NW equal warp ranges,
//     so every warp streams the same number of pages whatever the batch mix;
//   * each warp owns an NS-stage ring; lane 0 issues one TMA tile load per K or
//     V page slice (a (layer, page, kv head) slice is a contiguous 16 x hd run;
//     the arena is one 2-D tensor map of hd-element rows, SWIZZLE_128B, which
//     is exactly the XOR layout ldmatrix reads conflict free).  No per-16 B
//     address math, so issue never limits the stream;
//   * page-table entries of the next 32 pages are fetched one window ahead, one
//     lane per page, and the next segment's Q fragment is prefetched, so the
//     only round trips on a warp's critical path are the ring's own;
//   * pages that precede the current token were written by earlier steps, so
//     the ring fills before griddepcontrol.wait (the QKV GEMM is still running);
//     the CTA triggers its own successor immediately: the Wo GEMM (104 KB smem)
//     co-resides and streams its weights while this kernel drains;
//   * a unit cut by a range boundary is finished by the last of its warps to
//     arrive (atomic counter), merging the partial (m, l, o) of its warps in
//     warp order -- deterministic for a given batch.
// Math per page: G query heads of the kv head are the rows of one m16n8k16
// tile (rows >= G zero), Q.K^T and P.V on the tensor cores, online softmax in
// fp32 (exp2 domain).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "attention.cuh"
#include "common.cuh"

namespace sw {
namespace {

constexpr int kPg = 16;  // tokens per page

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Byte offset of 16 B chunk `chunk` (0 .. HD/8) of key row `row` inside one
// 16-row page slice as TMA SWIZZLE_128B lays it down: the slice is HD/64
// column halves of [16 rows][128 B], chunk index XOR (row & 7) inside a half.
template <int HD>
__device__ __forceinline__ uint32_t sw_off(int row, int chunk) {
    return static_cast<uint32_t>((chunk >> 3) * (kPg * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}

// Flat page index -> (row, kv head, page of the row).  pre[r] = sum of
// pages(r') for r' < r (n_rows + 1 entries in smem).
struct PageLoc {
    int row, hk, pg, np;
};
__device__ __forceinline__ PageLoc locate(const int* pre, int n_rows, int Hkv, long long f) {
    int lo = 0, hi = n_rows - 1;  // last row with pre[row] * Hkv <= f
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (static_cast<long long>(pre[mid]) * Hkv <= f) lo = mid;
        else hi = mid - 1;
    }
    const int np = pre[lo + 1] - pre[lo];
    const long long rem = f - static_cast<long long>(pre[lo]) * Hkv;
    const int hk = static_cast<int>(rem / np);
    return {lo, hk, static_cast<int>(rem - static_cast<long long>(hk) * np), np};
}

__device__ __forceinline__ long long range_start(long long w, long long W, long long NW) { return w * W / NW; }
// the warp whose range holds flat page f: max w with range_start(w) <= f
__device__ __forceinline__ long long warp_of(long long f, long long W, long long NW) {
    return ((f + 1) * NW - 1) / W;
}

template <int HD, int G, int NWARP, int NS>
struct FlatCfg {
    static constexpr int kSlice = kPg * HD * 2;  // bytes of one K or V page slice
    static constexpr int kStage = 2 * kSlice;
    static constexpr int kRing = NWARP * NS * kStage;
    // pre[rows + 1] | slot[rows] | ctx[rows], padded so the mbarriers stay 8 B aligned
    static constexpr int kPre = ((3 * kMaxDecodeRows + 1) * 4 + 15) / 16 * 16;
    static constexpr int kSmem = 1024 + kRing + kPre + NWARP * NS * 8;
};

template <int HD, int G, int NWARP, int NS>
__global__ void __launch_bounds__(NWARP * 32)
    attn_decode_flat_kernel(const __grid_constant__ CUtensorMap tm_kv, const kv_t* __restrict__ q,
                            __nv_bfloat16* __restrict__ out, DecodeFlatArgs a) {
    using C = FlatCfg<HD, G, NWARP, NS>;
    static_assert(G <= 8, "query rows live in the first 8 mma rows");
    static_assert(HD % 64 == 0, "head_dim: multiple of 64 (128 B swizzle halves)");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    int* pre = reinterpret_cast<int*>(smem + C::kRing);
    int* s_slot = pre + kMaxDecodeRows + 1;
    int* s_ctx = s_slot + kMaxDecodeRows;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kRing + C::kPre);

    griddep_launch_dependents();  // the successor GEMM co-resides and prefetches its weights
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const StepMeta* meta = a.meta;
    const int n_rows = meta->n;  // host-written before the step's first kernel
    const int Hkv = a.Hkv;
    // ---- page prefix over rows (block scan, 32 rows per pass)
    if (warp == 0) {
        int carry = 0;
        for (int r0 = 0; r0 < n_rows; r0 += 32) {
            const int r = r0 + lane;
            const int ctx_r = r < n_rows ? meta->pos[r] + 1 : 0;
            if (r < n_rows) {
                s_ctx[r] = ctx_r;
                s_slot[r] = meta->slot[r];
            }
            int v = (ctx_r + kPg - 1) / kPg;  // pages of the row's context
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            if (r < n_rows) pre[r + 1] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
        if (lane == 0) pre[0] = 0;
    }
    uint64_t* full = bars + warp * NS;
    if (lane == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        if (warp == 0) tma_prefetch_desc(&tm_kv);
    }
    __syncthreads();
    if (n_rows == 0) return;
    const long long W = static_cast<long long>(pre[n_rows]) * Hkv;
    // at most one warp per page, so every warp below NW owns >= 1 page (the
    // merge counts the warps of a unit as a contiguous id range)
    const long long NW = min(static_cast<long long>(gridDim.x) * NWARP, W);
    const long long gw = static_cast<long long>(blockIdx.x) * NWARP + warp;
    const long long f0 = range_start(gw, W, NW), f1 = range_start(gw + 1, W, NW);
    const int n_my = gw < NW ? static_cast<int>(f1 - f0) : 0;
    if (n_my == 0) {
        griddep_wait();
        return;
    }
    uint8_t* ring = smem + warp * NS * C::kStage;
    const uint64_t pol = l2_policy_evict_first();
    const int r = lane >> 2;

    // ---- page-id windows: lane j holds the page id and kv-head row offset of
    // relative page 32*win + j and whether it is the last page of its unit (its
    // KV may be written by this step).  The page-table load is consumed only
    // when the window is used, 32 pages later.
    struct Win {
        int pid, hrow;
        bool last;
    };
    auto window = [&](int win, Win& wv) {
        const int k = 32 * win + lane;
        wv.pid = 0;
        wv.hrow = 0;
        wv.last = false;
        if (k < n_my) {
            const PageLoc L = locate(pre, n_rows, Hkv, f0 + k);
            wv.pid = a.page_table[static_cast<long long>(s_slot[L.row]) * a.max_pages + L.pg];
            wv.hrow = L.hk * kPg;
            wv.last = L.pg == L.np - 1;
        }
    };
    auto issue = [&](int k, const Win& wv) {  // relative page k (its window is wv)
        const int kr = a.layer_row0 + __shfl_sync(0xffffffffu, wv.pid, k & 31) * a.page_rows +
                       __shfl_sync(0xffffffffu, wv.hrow, k & 31);
        if (lane == 0) {
            const int s = k % NS;
            uint8_t* dst = ring + s * C::kStage;
            fence_proxy_async_smem();  // generic-proxy reads/writes of the stage precede the refill
            mbar_expect_tx(&full[s], C::kStage);
#pragma unroll
            for (int h = 0; h < HD / 64; ++h) {
                tma_load_2d(dst + h * kPg * 128, &tm_kv, &full[s], h * 64, kr, pol);
                tma_load_2d(dst + C::kSlice + h * kPg * 128, &tm_kv, &full[s], h * 64, kr + a.v_rows, pol);
            }
        }
    };
    Win wcur, wnxt;
    window(0, wcur);
    int win_cur = 0;
    // ring fill before the predecessor finishes: pages written by earlier steps
    int issued = 0;
    {
        const unsigned stop = __ballot_sync(0xffffffffu, wcur.last);
        const int first_last = stop ? __ffs(stop) - 1 : 32;
        const int pre_n = min(min(NS, n_my), first_last);
        for (; issued < pre_n; ++issued) issue(issued, wcur);
    }
    griddep_wait();  // q, this step's K/V entries and page installs are visible from here
    if (issued < min(NS, n_my)) window(0, wcur);  // ids read early may predate the page install
    window(1, wnxt);
    for (; issued < min(NS, n_my); ++issued) issue(issued, wcur);  // NS <= 32: window 0

    // Q fragments (A operand rows = the G query heads); the next unit's are
    // fetched when a segment starts, so a segment switch never waits on them
    auto fetch_q = [&](int row, int hk, uint32_t (&dst)[HD / 16][2]) {
        const kv_t* qrow = q + static_cast<long long>(row) * a.H * HD + static_cast<long long>(hk * G + r) * HD;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            const int c = ks * 16 + (lane & 3) * 2;
            dst[ks][0] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c) : 0u;
            dst[ks][1] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c + 8) : 0u;
        }
    };
    PageLoc L = locate(pre, n_rows, Hkv, f0);
    int ctx = s_ctx[L.row];
    uint32_t qraw[HD / 16][2], qnext[HD / 16][2];
    uint32_t qf[HD / 16][4];
    auto set_q = [&]() {
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            qf[ks][0] = qraw[ks][0];
            qf[ks][1] = 0u;
            qf[ks][2] = qraw[ks][1];
            qf[ks][3] = 0u;
        }
    };
    auto prefetch_next = [&]() {
        int nh = L.hk + 1, nr = L.row;
        if (nh == Hkv) {
            nh = 0;
            ++nr;
        }
        if (nr < n_rows) fetch_q(nr, nh, qnext);
    };
    fetch_q(L.row, L.hk, qraw);
    set_q();
    prefetch_next();
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    bool seg_first = true;       // the segment starts at this warp's range start
    bool seg_whole = L.pg == 0;  // the segment starts at its unit's first page
    const uint32_t ring_addr = smem_addr(ring);

    for (int k = 0; k < n_my; ++k) {
        const int s = k % NS;
        mbar_wait(&full[s], (k / NS) & 1);
        const uint32_t kb = ring_addr + s * C::kStage;
        const uint32_t vb = kb + C::kSlice;
        const int valid = min(kPg, ctx - L.pg * kPg);
        if (valid < kPg) {  // stale rows past the context: zero V so 0 * garbage stays 0
            for (int i = lane; i < (kPg - valid) * (HD / 8); i += 32) {
                const int row = valid + i / (HD / 8), ch = i % (HD / 8);
                asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(vb + sw_off<HD>(row, ch)), "r"(0u)
                             : "memory");
            }
            __syncwarp();
        }
        // S = Q K^T over the page's 16 keys
        float sc[2][4];
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
            uint32_t b[4];
            const int key = (lane & 7) + ((lane >> 4) << 3);
            ldsm_x4(b, kb + sw_off<HD>(key, ks * 2 + ((lane >> 3) & 1)));
            mma_f16(sc[0], qf[ks], b[0], b[1]);
            mma_f16(sc[1], qf[ks], b[2], b[3]);
        }
        float mx = -INFINITY;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int key = nb * 8 + (lane & 3) * 2 + e;
                const float v = key < valid ? sc[nb][e] * a.scale_log2 : -INFINITY;
                sc[nb][e] = v;
                mx = fmaxf(mx, v);
            }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);  // finite: key 0 of every page is valid
        const float alpha = fast_exp2(m_run - m_new);
        m_run = m_new;
        float rs = 0.f;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
            sc[nb][0] = fast_exp2(sc[nb][0] - m_new);
            sc[nb][1] = fast_exp2(sc[nb][1] - m_new);
            rs += sc[nb][0] + sc[nb][1];
        }
        l_run = l_run * alpha + rs;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= alpha;
            o[i][1] *= alpha;
        }
        uint32_t pa[4];
        pa[0] = pack_h2(sc[0][0], sc[0][1]);
        pa[1] = 0u;
        pa[2] = pack_h2(sc[1][0], sc[1][1]);
        pa[3] = 0u;
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
            uint32_t b[4];
            const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
            ldsm_x4_t(b, vb + sw_off<HD>(key, dp * 2 + (lane >> 4)));
            mma_f16(o[2 * dp], pa, b[0], b[1]);
            mma_f16(o[2 * dp + 1], pa, b[2], b[3]);
        }
        __syncwarp();  // the stage's reads are done before it is refilled
        const int kn = k + NS;
        if (kn < n_my) {
            if ((kn >> 5) != win_cur) {  // advance the page-id windows
                wcur = wnxt;
                ++win_cur;
                window(win_cur + 1, wnxt);
            }
            issue(kn, wcur);
        }

        // ---- segment end: the unit's last page or the range's last page
        const bool unit_end = L.pg == L.np - 1;
        if (unit_end || k == n_my - 1) {
            float l_tot = l_run;
            l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 1);
            l_tot += __shfl_xor_sync(0xffffffffu, l_tot, 2);
            const long long unit = static_cast<long long>(L.row) * Hkv + L.hk;
            if (seg_whole && unit_end) {
                if (r < G) {
                    const float inv = 1.f / l_tot;
                    __nv_bfloat16* dst = out + static_cast<long long>(L.row) * a.H * HD +
                                         static_cast<long long>(L.hk * G + r) * HD + (lane & 3) * 2;
#pragma unroll
                    for (int i = 0; i < HD / 8; ++i)
                        *reinterpret_cast<uint32_t*>(dst + i * 8) = pack_bf2(o[i][0] * inv, o[i][1] * inv);
                }
            } else {
                // partial (m, l, unnormalised o) of this warp for the unit; slot 0 = the
                // segment that starts the warp's range, 1 = the one that ends it
                const long long slot = gw * 2 + (seg_first ? 0 : 1);
                if (r < G) {
                    float* po = a.part_o + (slot * G + r) * HD + (lane & 3) * 2;
#pragma unroll
                    for (int i = 0; i < HD / 8; ++i)
                        __stcg(reinterpret_cast<float2*>(po + i * 8), make_float2(o[i][0], o[i][1]));
                    if ((lane & 3) == 0)
                        __stcg(reinterpret_cast<float2*>(a.part_ml + (slot * G + r) * 2), make_float2(m_run, l_tot));
                }
                __syncwarp();  // every lane's partial stores happen-before lane 0's release below
                const long long u0 = static_cast<long long>(pre[L.row]) * Hkv + static_cast<long long>(L.hk) * L.np;
                const long long ca = warp_of(u0, W, NW), cb = warp_of(u0 + L.np - 1, W, NW);
                unsigned last = 0;
                if (lane == 0) {
                    last = atomic_add_acq_rel_gpu(a.counters + unit, 1u) == static_cast<unsigned>(cb - ca);
                    if (last) a.counters[unit] = 0u;
                }
                last = __shfl_sync(0xffffffffu, last, 0);  // lane 0's acquire, ordered to the warp
                if (last) {
                    // merge the unit's partials in warp order (online rescale, one pass); each
                    // lane owns PER contiguous floats of the [G][HD] tile, loads for NB
                    // contributors in flight together
                    constexpr int PER = G * HD / 32;
                    static_assert(PER % 4 == 0, "vector merge");
                    const int e0 = lane * PER, g = e0 / HD;
                    const bool shifted = range_start(ca, W, NW) < u0;  // the unit is not warp ca's first segment
                    float Mx = -INFINITY, Ls = 0.f, Os[PER];
#pragma unroll
                    for (int qq = 0; qq < PER; ++qq) Os[qq] = 0.f;
                    constexpr int NB = PER <= 8 ? 4 : 2;  // contributors per batch (register budget)
                    for (long long c0 = ca; c0 <= cb; c0 += NB) {
                        float2 ml[NB];
                        float4 ov[NB][PER / 4];
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            const long long c = c0 + j;
                            if (c <= cb) {
                                const long long sl = c * 2 + ((c == ca && shifted) ? 1 : 0);
                                ml[j] = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (sl * G + g) * 2));
#pragma unroll
                                for (int v = 0; v < PER / 4; ++v)
                                    ov[j][v] = __ldcg(reinterpret_cast<const float4*>(a.part_o + sl * G * HD + e0) + v);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            if (c0 + j <= cb) {
                                const float mn = fmaxf(Mx, ml[j].x);
                                const float c_old = fast_exp2(Mx - mn), c_new = fast_exp2(ml[j].x - mn);
                                Mx = mn;
                                Ls = Ls * c_old + ml[j].y * c_new;
#pragma unroll
                                for (int v = 0; v < PER / 4; ++v) {
                                    Os[4 * v + 0] = Os[4 * v + 0] * c_old + ov[j][v].x * c_new;
                                    Os[4 * v + 1] = Os[4 * v + 1] * c_old + ov[j][v].y * c_new;
                                    Os[4 * v + 2] = Os[4 * v + 2] * c_old + ov[j][v].z * c_new;
                                    Os[4 * v + 3] = Os[4 * v + 3] * c_old + ov[j][v].w * c_new;
                                }
                            }
                        }
                    }
                    const float inv = 1.f / Ls;
                    uint32_t* dst = reinterpret_cast<uint32_t*>(out + static_cast<long long>(L.row) * a.H * HD +
                                                                static_cast<long long>(L.hk * G) * HD + e0);
#pragma unroll
                    for (int v = 0; v < PER / 4; ++v)
                        *reinterpret_cast<uint2*>(dst + 2 * v) =
                            make_uint2(pack_bf2(Os[4 * v] * inv, Os[4 * v + 1] * inv),
                                       pack_bf2(Os[4 * v + 2] * inv, Os[4 * v + 3] * inv));
                }
            }
            // next segment
            if (k + 1 < n_my) {
                seg_first = false;
                L.pg = 0;
                if (++L.hk == Hkv) {
                    L.hk = 0;
                    ++L.row;
                    L.np = pre[L.row + 1] - pre[L.row];
                    ctx = s_ctx[L.row];
                }
                seg_whole = true;
#pragma unroll
                for (int ks = 0; ks < HD / 16; ++ks) {
                    qraw[ks][0] = qnext[ks][0];
                    qraw[ks][1] = qnext[ks][1];
                }
                set_q();
                prefetch_next();
#pragma unroll
                for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
                m_run = -INFINITY;
                l_run = 0.f;
            }
        } else {
            ++L.pg;
        }
    }
}

template <int HD, int G, int NWARP, int NS>
void flat_launch(const CUtensorMap& tm, const kv_t* q, __nv_bfloat16* out, const DecodeFlatArgs& a, int ctas,
                 cudaStream_t st) {
    using C = FlatCfg<HD, G, NWARP, NS>;
    static bool cfg = false;
    if (!cfg) {
        SW_CUDA(cudaFuncSetAttribute(attn_decode_flat_kernel<HD, G, NWARP, NS>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        SW_CUDA(cudaFuncSetAttribute(attn_decode_flat_kernel<HD, G, NWARP, NS>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
        cfg = true;
    }
    launch_k(attn_decode_flat_kernel<HD, G, NWARP, NS>, dim3(ctas), dim3(NWARP * 32), C::kSmem, st, tm, q, out, a);
}

// Ring shape: warps per CTA x stages per warp, and CTAs per SM (SW_ATTN_FLAT_CFG
// = "warps,stages,ctas_per_sm"; tuning only).
struct FlatShape {
    int warps, stages, per_sm;
};
FlatShape flat_shape(int hd) {
    static const FlatShape env = [] {
        FlatShape f{0, 0, 0};
        if (const char* v = std::getenv("SW_ATTN_FLAT_CFG")) std::sscanf(v, "%d,%d,%d", &f.warps, &f.stages, &f.per_sm);
        return f;
    }();
    if (env.warps) return env;
    // measured (profiles/r01c/attn_flat_sweep.txt): Llama-1B (hd 64) one 8-warp CTA per SM, 4 pages
    // per warp in flight; Llama-8B (hd 128) two 4-warp CTAs per SM, double-buffered -- both leave
    // room for the successor GEMM's CTA on the SM
    return hd == 64 ? FlatShape{8, 4, 1} : FlatShape{4, 2, 2};
}

template <int HD, int G>
void flat_dispatch(const CUtensorMap& tm, const kv_t* q, __nv_bfloat16* out, const DecodeFlatArgs& a,
                   int sms, cudaStream_t st) {
    const FlatShape f = flat_shape(HD);
    const int ctas = sms * std::max(1, f.per_sm);
#define SW_FLAT(W, S)                                                   \
    if (f.warps == W && f.stages == S) {                               \
        flat_launch<HD, G, W, S>(tm, q, out, a, ctas, st);             \
        return;                                                        \
    }
    if constexpr (HD == 64) {
        SW_FLAT(4, 6) SW_FLAT(4, 4) SW_FLAT(8, 4) SW_FLAT(8, 6) SW_FLAT(8, 3)
    } else {
        SW_FLAT(4, 3) SW_FLAT(8, 3) SW_FLAT(8, 2) SW_FLAT(4, 2)
    }
#undef SW_FLAT
    throw_cuda("attn_decode_flat: unsupported ring shape", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace

size_t attn_decode_flat_part_rows(int sms) {
    // two partial slots per warp, <= 16 warps per SM over the ring shapes (rows of G x hd floats)
    return static_cast<size_t>(2) * 16 * sms;
}

void attn_decode_flat(const CUtensorMap& tm_kv, const kv_t* q, __nv_bfloat16* out, const DecodeFlatArgs& a,
                      int sms, int hd, int G, cudaStream_t st) {
    if (hd == 64 && G == 4) flat_dispatch<64, 4>(tm_kv, q, out, a, sms, st);
    else if (hd == 64 && G == 2) flat_dispatch<64, 2>(tm_kv, q, out, a, sms, st);
    else if (hd == 128 && G == 4) flat_dispatch<128, 4>(tm_kv, q, out, a, sms, st);
    else throw_cuda("attn_decode_flat: unsupported (head_dim, group)", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw

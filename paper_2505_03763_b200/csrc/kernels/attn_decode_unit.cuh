// Decode attention work unit of the per-unit split-KV kernel (attention.cu).
// (A persistent whole-step kernel also ran this unit; measured 2.8x slower than
// the per-projection kernels, profiles/r01c/step_check_persistent_vs_kernels.txt,
// and removed.)
//
// One unit = (row, kv head, split of the context), run by 128 threads (4
// warps).  The warps stream disjoint KB-key blocks of the split (warp w takes
// blocks w, w+4, ...) through private double-buffered smem, each with its own
// online softmax; the G query heads of the kv head are the rows of a 16-row
// mma tile (rows >= G are zero), so Q.K^T and P.V run on the tensor cores and
// the unit is a pure HBM stream of K/V pages.  Warps merge in smem; splits
// merge in the last-arriving unit of the (row, kv head), in split order, so
// the result does not depend on timing.
#pragma once

#include "attention.cuh"
#include "common.cuh"

namespace sw {
namespace attn {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const int sz = valid ? 16 : 0;  // zero-fill when invalid
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(smem)), "l"(gmem), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}

// [rows][HD] 16-bit tile, 16 B chunks XOR-swizzled by row.
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
    return row * HD + ((chunk ^ (row & 7)) << 3);
}

constexpr int kPage = 16;            // tokens per KV page (fixed: shifts, not divisions, in the address math)
constexpr int kPartSplits = 16;      // stride of the split-partial buffers (>= any split count)
constexpr int kMaxChunkPages = 512;  // page ids of one decode split staged in smem (8192 keys)
// keys per K/V block of a warp's ring: 16 at every head dim (hd 64 used 32: with 16, a warp of a
// short unit has twice the blocks to pipeline and the ring half the smem -- Llama-1B b=64 ctx 512
// step 0.992 -> 0.969 ms; profiles/r02s4/decode_attention_kb_ab.txt)
template <int HD>
constexpr int decode_kb() {
    return 16;
}
// dynamic smem of one unit runner (4 warps): per-warp NS-stage K/V rings + warp-merge scratch
template <int HD, int G, int NS = 2>
constexpr int decode_unit_smem() {
    return 4 * (2 * NS * decode_kb<HD>() * HD) * 2 + (8 * G + 4 * G * HD) * 4;
}

// Split plan of one row: how many units its context is cut into and the keys
// per unit (every split non-empty).  `want` = splits that would bring the
// step to its target unit count; `cap` = the most splits allowed.
struct SplitPlan {
    int splits, chunk;
};
template <int KB>
__device__ __forceinline__ SplitPlan decode_split_plan(int ctx, int want, int cap) {
    const int splits0 = max(cdiv(ctx, kMaxChunkPages * kPage), max(1, min(min(want, cap), cdiv(ctx, 4 * KB))));
    const int chunk = cdiv(cdiv(ctx, splits0), KB) * KB;
    return {cdiv(ctx, chunk), chunk};
}

// One unit.  `tid` in [0, 128); `sync()` synchronises exactly the 128
// threads running the unit.  smem: dsm (decode_unit_smem bytes), s_pages
// (kMaxChunkPages ints), s_last (one word).
// `wait_pred()` is called once, after the ring fill of key blocks older than this
// step's token (KV written by earlier steps, page ids installed earlier) and before
// anything the predecessor kernel produces (q, the new K/V entry, a page installed
// this step) is read: the unit's HBM stream starts while the QKV GEMM drains.
template <int HD, int G, int KB, int NS = 2, class Sync, class Wait>
__device__ __forceinline__ void decode_unit(const DecodeAttnArgs& a, const kv_t* __restrict__ q,
                                            const kv_t* __restrict__ kv_layer,
                                            __nv_bfloat16* __restrict__ out, int row, int hk, int split,
                                            const SplitPlan& plan, int ctx, uint8_t* dsm, int32_t* s_pages,
                                            uint32_t* s_last, int tid, Sync sync, Wait wait_pred) {
    static_assert(G <= 8, "query rows live in the first 8 mma rows");
    constexpr int CH = HD / 8;
    const int warp = tid >> 5, lane = tid & 31;
    kv_t* wK = reinterpret_cast<kv_t*>(dsm) + warp * (2 * NS * KB * HD);  // [NS][KB][HD]
    kv_t* wV = wK + NS * KB * HD;                                                  // [NS][KB][HD]
    float* cm = reinterpret_cast<float*>(dsm + 4 * (2 * NS * KB * HD) * 2);  // [4][G]
    float* cl = cm + 4 * G;                                             // [4][G]
    float* co = cl + 4 * G;                                             // [4][G][HD]
    const int splits = plan.splits;
    const int k_begin = split * plan.chunk;
    const int k_end = min(ctx, k_begin + plan.chunk);
    {  // this split's page ids -> smem (one read per page, not per 16 B chunk)
        const int32_t* ptab = a.page_table + static_cast<int64_t>(a.meta->slot[row]) * a.max_pages;
        const int p0 = k_begin / kPage, p1 = (k_end - 1) / kPage;
        for (int i = tid; i <= p1 - p0; i += 128) s_pages[i] = ptab[p0 + i];
    }
    const int page_base = k_begin / kPage;
    const int n_blocks = cdiv(k_end - k_begin, KB);

    // A block is KB / kPage whole pages (blocks start page aligned); a (layer,
    // page, kv head) K or V slice is one contiguous kPage x HD run, so lane l
    // copies 16 B chunks l, l + 32, ... of it: one page-id read and one base
    // address per page, the rest compile-time offsets (the generic per-chunk
    // index math made this kernel integer-issue bound, profiles/r01b).
    const char* kv_head = reinterpret_cast<const char*>(kv_layer + static_cast<int64_t>(hk) * kPage * HD);
    const int64_t page_bytes = a.page_stride * 2, v_off = a.kv_stride * 2;
    auto load = [&](int blk, int buf) {
        const int k0 = k_begin + blk * KB;
#pragma unroll
        for (int pg = 0; pg < KB / kPage; ++pg) {
            const int key0 = k0 + pg * kPage;
            const int page = key0 < k_end ? s_pages[key0 / kPage - page_base] : 0;
            const char* src = kv_head + static_cast<int64_t>(page) * page_bytes;
#pragma unroll
            for (int j = 0; j < kPage * CH / 32; ++j) {
                const int idx = lane + 32 * j;  // 16 B chunk of the page slice
                const int r = idx / CH, c = idx % CH;
                const bool ok = key0 + r < k_end;
                const int dst = swz<HD>(pg * kPage + r, c);
                cp_async16(wK + buf * KB * HD + dst, src + idx * 16, ok);
                cp_async16(wV + buf * KB * HD + dst, src + v_off + idx * 16, ok);
            }
        }
    };

    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;  // row r (c0/c1); rows r+8 are padding

    sync();  // s_pages
    // warp w streams blocks w, w + 4, ... through an NS-stage ring (NS - 1 in flight while one is computed)
    const int my_blocks = n_blocks > warp ? (n_blocks - warp + 3) / 4 : 0;
    // ring fill before the wait: blocks that end before this step's token (the last key, ctx - 1) --
    // in issue order, one commit per slot exactly as the in-order fill would make them
    int filled = 0;
#pragma unroll
    for (int i = 0; i < NS - 1; ++i) {
        const bool old_block = k_begin + (warp + 4 * i + 1) * KB < ctx;  // ends before key ctx - 1
        if (filled == i && (i >= my_blocks || old_block)) {
            if (i < my_blocks) load(warp + 4 * i, i);
            cp_async_commit();
            ++filled;
        }
    }
    wait_pred();
    if (k_end == ctx) {  // this split holds the token's page: its id may have been installed by this step
        sync();
        if (tid == 0) {
            const int32_t* ptab = a.page_table + static_cast<int64_t>(a.meta->slot[row]) * a.max_pages;
            s_pages[(ctx - 1) / kPage - page_base] = ptab[(ctx - 1) / kPage];
        }
        sync();
    }
#pragma unroll
    for (int i = 0; i < NS - 1; ++i) {
        if (i >= filled) {
            if (i < my_blocks) load(warp + 4 * i, i);
            cp_async_commit();
        }
    }
    // Q fragment (A operand, rows = query heads of this kv head)
    const int r = lane >> 2;
    uint32_t qf[HD / 16][4];
    const kv_t* qrow = q + static_cast<int64_t>(row) * a.H * HD + static_cast<int64_t>(hk * G + r) * HD;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
        const int c = ks * 16 + (lane & 3) * 2;
        qf[ks][0] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c) : 0u;
        qf[ks][1] = 0u;
        qf[ks][2] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c + 8) : 0u;
        qf[ks][3] = 0u;
    }


    for (int it = 0; it < my_blocks; ++it) {
        const int blk = warp + 4 * it;
        const int buf = it % NS;
        if (it + NS - 1 < my_blocks) load(blk + 4 * (NS - 1), (it + NS - 1) % NS);
        cp_async_commit();
        cp_async_wait<NS - 1>();
        __syncwarp();
        const kv_t* K = wK + buf * KB * HD;
        const kv_t* V = wV + buf * KB * HD;
        float sc[KB / 8][4];
#pragma unroll
        for (int nb = 0; nb < KB / 8; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
            for (int np = 0; np < KB / 16; ++np) {
                uint32_t b[4];
                const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int c = ks * 2 + ((lane >> 3) & 1);
                ldsm_x4(b, K + swz<HD>(key, c));
                mma_f16(sc[2 * np], qf[ks], b[0], b[1]);
                mma_f16(sc[2 * np + 1], qf[ks], b[2], b[3]);
            }
        }
        const int kbase = k_begin + blk * KB;
        float mx = -INFINITY;
#pragma unroll
        for (int nb = 0; nb < KB / 8; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int key = kbase + nb * 8 + (lane & 3) * 2 + e;
                const float v = key < k_end ? sc[nb][e] * a.scale_log2 : -INFINITY;
                sc[nb][e] = v;
                mx = fmaxf(mx, v);
            }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);  // finite: the block's first key is valid
        const float alpha = fast_exp2(m_run - m_new);
        m_run = m_new;
        float rs = 0.f;
#pragma unroll
        for (int nb = 0; nb < KB / 8; ++nb) {
            sc[nb][0] = fast_exp2(sc[nb][0] - m_new);
            sc[nb][1] = fast_exp2(sc[nb][1] - m_new);
            sc[nb][2] = sc[nb][3] = 0.f;  // padding rows
            rs += sc[nb][0] + sc[nb][1];
        }
        l_run = l_run * alpha + rs;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= alpha;
            o[i][1] *= alpha;
        }
#pragma unroll
        for (int kk = 0; kk < KB / 16; ++kk) {
            uint32_t pa[4];
            pa[0] = pack_h2(sc[2 * kk][0], sc[2 * kk][1]);
            pa[1] = 0u;
            pa[2] = pack_h2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
            pa[3] = 0u;
#pragma unroll
            for (int dp = 0; dp < HD / 16; ++dp) {
                uint32_t b[4];
                const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dp * 2 + (lane >> 4);
                ldsm_x4_t(b, V + swz<HD>(key, c));
                mma_f16(o[2 * dp], pa, b[0], b[1]);
                mma_f16(o[2 * dp + 1], pa, b[2], b[3]);
            }
        }
        __syncwarp();
    }
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    // ---- merge the 4 warps
    if (r < G) {
        if ((lane & 3) == 0) {
            cm[warp * G + r] = m_run;
            cl[warp * G + r] = l_run;
        }
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            float* dst = co + (warp * G + r) * HD + i * 8 + (lane & 3) * 2;
            dst[0] = o[i][0];
            dst[1] = o[i][1];
        }
    }
    sync();
    const int64_t pidx = (static_cast<int64_t>(row) * a.Hkv + hk) * kPartSplits + split;
    for (int idx = tid; idx < G * HD; idx += 128) {
        const int g = idx / HD, d = idx % HD;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, cm[w * G + g]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float sc_w = cm[w * G + g] == -INFINITY ? 0.f : fast_exp2(cm[w * G + g] - M);
            L += cl[w * G + g] * sc_w;
            O += co[(w * G + g) * HD + d] * sc_w;
        }
        if (splits == 1) {
            out[static_cast<int64_t>(row) * a.H * HD + (hk * G + g) * HD + d] = __float2bfloat16_rn(O / L);
        } else {
            __stcg(a.part_o + pidx * G * HD + idx, O);
            if (d == 0) {
                __stcg(a.part_ml + (pidx * G + g) * 2, M);
                __stcg(a.part_ml + (pidx * G + g) * 2 + 1, L);
            }
        }
    }
    if (splits == 1) {
        sync();  // cm/cl/co and s_pages are reused by the runner's next unit
        return;
    }
    // ---- last split to arrive merges all splits in order (the barrier orders every thread's
    // partial stores before thread 0's release; its acquire reaches the others through the next one)
    sync();
    if (tid == 0) {
        unsigned* cnt = a.counters + static_cast<int64_t>(row) * a.Hkv + hk;
        *s_last = atomic_add_acq_rel_gpu(cnt, 1u) == static_cast<unsigned>(splits - 1);
        if (*s_last) *cnt = 0u;
    }
    sync();
    if (*s_last) {
        const int64_t base = (static_cast<int64_t>(row) * a.Hkv + hk) * kPartSplits;
        for (int idx = tid; idx < G * HD; idx += 128) {
            const int g = idx / HD;
            float M = -INFINITY;
            for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(a.part_ml + ((base + sp) * G + g) * 2));
            float L = 0.f, O = 0.f;
            for (int sp = 0; sp < splits; ++sp) {
                const float w = fast_exp2(__ldcg(a.part_ml + ((base + sp) * G + g) * 2) - M);
                L += __ldcg(a.part_ml + ((base + sp) * G + g) * 2 + 1) * w;
                O += __ldcg(a.part_o + (base + sp) * G * HD + idx) * w;
            }
            out[static_cast<int64_t>(row) * a.H * HD + (hk * G) * HD + idx] = __float2bfloat16_rn(O / L);
        }
    }
    sync();  // s_last / smem reuse
}

}  // namespace attn
}  // namespace sw

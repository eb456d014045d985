// Attention over the paged KV cache.
//
// Prefill: causal flash attention (online softmax, fp32 statistics) for a
//   varlen batch of prompts, GQA.  One CTA = 64 query rows of one head of one
//   prompt (4 warps x 16 rows); K/V stream through smem in 64-key blocks read
//   straight from the 16-token pages just written by rope_kv (double-buffered
//   cp.async, XOR-swizzled 16 B chunks for conflict-free ldmatrix); QK^T and
//   PV on the tensor cores with mma.m16n8k16 bf16 -> fp32.
// Decode: split-KV paged attention on the tensor cores (see below); the G =
//   H/Hkv query heads sharing a kv head are packed into one mma tile so every
//   K/V byte is read once per step.  HBM-bound by design.
#include <algorithm>

#include "attention.cuh"
#include "common.cuh"

namespace sw {

namespace {

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
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// [rows][HD] bf16 tile, 16 B chunks XOR-swizzled by row.
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
    return row * HD + ((chunk ^ (row & 7)) << 3);
}

constexpr int kQRows = 64;
constexpr int kKeys = 64;
constexpr int kPage = 16;        // tokens per KV page (fixed: shifts, not divisions, in the address math)
constexpr int kPartSplits = 16;  // stride of the split-partial buffers (>= any grid x)
constexpr int kMaxChunkPages = 512;  // page ids of one decode split staged in smem (8192 keys)

template <int HD>
__global__ void __launch_bounds__(128) attn_prefill_kernel(const __nv_bfloat16* __restrict__ q,
                                                           const __nv_bfloat16* __restrict__ kv_layer,
                                                           __nv_bfloat16* __restrict__ out, PrefillAttnArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
    __nv_bfloat16* sK = sQ + kQRows * HD;       // [2][64][HD]
    __nv_bfloat16* sV = sK + 2 * kKeys * HD;    // [2][64][HD]
    constexpr int CH = HD / 8;                  // 16 B chunks per row

    const int tile = blockIdx.x;
    if (tile >= *a.n_tiles) return;
    const int h = blockIdx.y;
    const int hk = h / (a.H / a.Hkv);
    const int s = a.tile_seq[tile];
    const int q0 = a.tile_q0[tile];
    const int start = a.cu_seqlens[s];
    const int len = a.cu_seqlens[s + 1] - start;
    const int slot = a.seq_slot[s];
    const int32_t* ptab = a.page_table + static_cast<int64_t>(slot) * a.max_pages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t qstride = static_cast<int64_t>(a.H) * HD;

    // Q tile -> smem (zero rows past the prompt)
    for (int i = tid; i < kQRows * CH; i += 128) {
        const int r = i / CH, c = i % CH;
        const bool ok = q0 + r < len;
        const __nv_bfloat16* src = q + (start + (ok ? q0 + r : 0)) * qstride + h * HD + c * 8;
        cp_async16(sQ + swz<HD>(r, c), src, ok);
    }
    auto load_kv = [&](int blk, int buf) {
        for (int i = tid; i < kKeys * CH; i += 128) {
            const int r = i / CH, c = i % CH;
            const int key = blk * kKeys + r;
            const bool ok = key < len;
            const int page = ok ? ptab[key / kPage] : 0;
            const __nv_bfloat16* base = kv_layer + static_cast<int64_t>(page) * a.page_stride +
                                        static_cast<int64_t>(hk) * kPage * HD +
                                        static_cast<int64_t>(key % kPage) * HD + c * 8;
            cp_async16(sK + buf * kKeys * HD + swz<HD>(r, c), base, ok);
            cp_async16(sV + buf * kKeys * HD + swz<HD>(r, c), base + a.kv_stride, ok);
        }
    };
    const int last_blk = min((q0 + kQRows - 1) / kKeys, (len - 1) / kKeys);
    load_kv(0, 0);
    cp_async_commit();

    uint32_t qf[HD / 16][4];
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    const int row_a = q0 + warp * 16 + (lane >> 2);  // query position of c0/c1; +8 for c2/c3

    for (int blk = 0; blk <= last_blk; ++blk) {
        const int buf = blk & 1;
        if (blk < last_blk) {
            load_kv(blk + 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (blk == 0) {
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks) {
                const int r = warp * 16 + (lane & 15);
                const int c = ks * 2 + (lane >> 4);
                ldsm_x4(qf[ks], sQ + swz<HD>(r, c));
            }
        }
        const __nv_bfloat16* K = sK + buf * kKeys * HD;
        const __nv_bfloat16* V = sV + buf * kKeys * HD;
        float sc[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t b[4];
                const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
                const int c = ks * 2 + ((lane >> 3) & 1);
                ldsm_x4(b, K + swz<HD>(key, c));
                mma_bf16(sc[2 * np], qf[ks], b[0], b[1]);
                mma_bf16(sc[2 * np + 1], qf[ks], b[2], b[3]);
            }
        }
        // mask + online softmax (log2 domain)
        const bool edge = (blk + 1) * kKeys > q0 || (blk + 1) * kKeys > len;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = sc[nb][e] * a.scale_log2;
                if (edge) {
                    const int key = blk * kKeys + nb * 8 + (lane & 3) * 2 + (e & 1);
                    const int qp = row_a + ((e >> 1) << 3);
                    if (key > qp || key >= len) v = -INFINITY;
                }
                sc[nb][e] = v;
                mx[e >> 1] = fmaxf(mx[e >> 1], v);
            }
        }
        float alpha[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
            const float m_new = fmaxf(m_run[r], mx[r]);
            const float m_use = m_new == -INFINITY ? 0.f : m_new;
            alpha[r] = exp2f(m_run[r] - m_use);
            m_run[r] = m_new;
            mx[r] = m_use;
        }
        float rs[2] = {0.f, 0.f};
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float p = exp2f(sc[nb][e] - mx[e >> 1]);
                sc[nb][e] = p;
                rs[e >> 1] += p;
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * alpha[r] + rs[r];
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= alpha[0];
            o[i][1] *= alpha[0];
            o[i][2] *= alpha[1];
            o[i][3] *= alpha[1];
        }
        // O += P V
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4];
            pa[0] = pack_bf2(sc[2 * kk][0], sc[2 * kk][1]);
            pa[1] = pack_bf2(sc[2 * kk][2], sc[2 * kk][3]);
            pa[2] = pack_bf2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
            pa[3] = pack_bf2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
            for (int dp = 0; dp < HD / 16; ++dp) {
                uint32_t b[4];
                const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dp * 2 + (lane >> 4);
                ldsm_x4_t(b, V + swz<HD>(key, c));
                mma_bf16(o[2 * dp], pa, b[0], b[1]);
                mma_bf16(o[2 * dp + 1], pa, b[2], b[3]);
            }
        }
        __syncthreads();
    }
    // normalise + store (row sums were kept per thread: reduce over the quad)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
        l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int qp = row_a + r * 8;
        if (qp >= len) continue;
        const float inv = 1.f / l_run[r];
        __nv_bfloat16* dst = out + (start + qp) * qstride + h * HD + (lane & 3) * 2;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i)
            *reinterpret_cast<uint32_t*>(dst + i * 8) = pack_bf2(o[i][2 * r] * inv, o[i][2 * r + 1] * inv);
    }
}

// ------------------------------------------------------------------ decode
// One CTA = (row, kv head, split of the context).  Its 4 warps stream
// disjoint KB-key blocks of the split (warp w takes blocks w, w+4, ...)
// through private double-buffered smem, each with its own online softmax;
// the G query heads of the kv head are the rows of a 16-row mma tile
// (rows >= G are zero), so Q.K^T and P.V run on the tensor cores and the
// kernel is a pure HBM stream of K/V pages.  Warps merge in smem; splits
// merge in the last-arriving CTA of the (row, kv head) (ordered, so results
// do not depend on timing).
template <int HD, int G, int KB>
__global__ void __launch_bounds__(128) attn_decode_kernel(const __nv_bfloat16* __restrict__ q,
                                                          const __nv_bfloat16* __restrict__ kv_layer,
                                                          __nv_bfloat16* __restrict__ out, DecodeAttnArgs a) {
    static_assert(G <= 8, "query rows live in the first 8 mma rows");
    constexpr int CH = HD / 8;
    extern __shared__ __align__(128) uint8_t dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __nv_bfloat16* wK = reinterpret_cast<__nv_bfloat16*>(dsm) + warp * (4 * KB * HD);  // [2][KB][HD]
    __nv_bfloat16* wV = wK + 2 * KB * HD;                                               // [2][KB][HD]
    float* cm = reinterpret_cast<float*>(dsm + 4 * (4 * KB * HD) * 2);  // [4][G]
    float* cl = cm + 4 * G;                                             // [4][G]
    float* co = cl + 4 * G;                                             // [4][G][HD]
    __shared__ uint32_t s_last;

    __shared__ int32_t s_pages[kMaxChunkPages];
    griddep_launch_dependents();
    griddep_wait();
    const int n_rows = a.meta->n;
    const int row = blockIdx.z;
    if (row >= n_rows) return;
    const int ctx = a.meta->pos[row] + 1;
    // splits chosen at run time: only as many as it takes to reach
    // a.target_ctas CTAs, each warp keeping >= 1 key block
    const int want = cdiv(a.target_ctas, n_rows * a.Hkv);
    const int splits0 = max(cdiv(ctx, kMaxChunkPages * kPage),
                            max(1, min(min(want, static_cast<int>(gridDim.x)), cdiv(ctx, 4 * KB))));
    const int chunk = cdiv(cdiv(ctx, splits0), KB) * KB;
    const int splits = cdiv(ctx, chunk);  // every split non-empty
    const int split = blockIdx.x;
    if (split >= splits) return;
    const int k_begin = split * chunk;
    const int k_end = min(ctx, k_begin + chunk);
    if (k_begin >= k_end) return;
    const int hk = blockIdx.y;
    {  // this split's page ids -> smem (one read per page, not per 16 B chunk)
        const int32_t* ptab = a.page_table + static_cast<int64_t>(a.meta->slot[row]) * a.max_pages;
        const int p0 = k_begin / kPage, p1 = (k_end - 1) / kPage;
        for (int i = threadIdx.x; i <= p1 - p0; i += 128) s_pages[i] = ptab[p0 + i];
    }
    const int page_base = k_begin / kPage;
    const int n_blocks = cdiv(k_end - k_begin, KB);

    // Q fragment (A operand, rows = query heads of this kv head)
    const int r = lane >> 2;
    uint32_t qf[HD / 16][4];
    const __nv_bfloat16* qrow = q + static_cast<int64_t>(row) * a.H * HD + static_cast<int64_t>(hk * G + r) * HD;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
        const int c = ks * 16 + (lane & 3) * 2;
        qf[ks][0] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c) : 0u;
        qf[ks][1] = 0u;
        qf[ks][2] = r < G ? *reinterpret_cast<const uint32_t*>(qrow + c + 8) : 0u;
        qf[ks][3] = 0u;
    }

    auto load = [&](int blk, int buf) {
        const int k0 = k_begin + blk * KB;
        for (int i = lane; i < KB * CH; i += 32) {
            const int kr = i / CH, c = i % CH;
            const int key = k0 + kr;
            const bool ok = key < k_end;
            const int page = ok ? s_pages[key / kPage - page_base] : 0;
            const __nv_bfloat16* src = kv_layer + static_cast<int64_t>(page) * a.page_stride +
                                       static_cast<int64_t>(hk) * kPage * HD +
                                       static_cast<int64_t>(key % kPage) * HD + c * 8;
            cp_async16(wK + buf * KB * HD + swz<HD>(kr, c), src, ok);
            cp_async16(wV + buf * KB * HD + swz<HD>(kr, c), src + a.kv_stride, ok);
        }
    };

    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;  // row r (c0/c1); rows r+8 are padding

    __syncthreads();  // s_pages
    int it = 0;
    if (warp < n_blocks) {
        load(warp, 0);
        cp_async_commit();
    }
    for (int blk = warp; blk < n_blocks; blk += 4, ++it) {
        const int buf = it & 1;
        if (blk + 4 < n_blocks) {
            load(blk + 4, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const __nv_bfloat16* K = wK + buf * KB * HD;
        const __nv_bfloat16* V = wV + buf * KB * HD;
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
                mma_bf16(sc[2 * np], qf[ks], b[0], b[1]);
                mma_bf16(sc[2 * np + 1], qf[ks], b[2], b[3]);
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
        const float alpha = exp2f(m_run - m_new);
        m_run = m_new;
        float rs = 0.f;
#pragma unroll
        for (int nb = 0; nb < KB / 8; ++nb) {
            sc[nb][0] = exp2f(sc[nb][0] - m_new);
            sc[nb][1] = exp2f(sc[nb][1] - m_new);
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
            pa[0] = pack_bf2(sc[2 * kk][0], sc[2 * kk][1]);
            pa[1] = 0u;
            pa[2] = pack_bf2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
            pa[3] = 0u;
#pragma unroll
            for (int dp = 0; dp < HD / 16; ++dp) {
                uint32_t b[4];
                const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
                const int c = dp * 2 + (lane >> 4);
                ldsm_x4_t(b, V + swz<HD>(key, c));
                mma_bf16(o[2 * dp], pa, b[0], b[1]);
                mma_bf16(o[2 * dp + 1], pa, b[2], b[3]);
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
    __syncthreads();
    const int64_t pidx = (static_cast<int64_t>(row) * a.Hkv + hk) * kPartSplits + split;
    for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
        const int g = idx / HD, d = idx % HD;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, cm[w * G + g]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float sc_w = cm[w * G + g] == -INFINITY ? 0.f : exp2f(cm[w * G + g] - M);
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
    if (splits == 1) return;
    // ---- last split to arrive merges all splits in order
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* cnt = a.counters + static_cast<int64_t>(row) * a.Hkv + hk;
        s_last = atomicAdd(cnt, 1u) == static_cast<unsigned>(splits - 1);
        if (s_last) *cnt = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int64_t base = (static_cast<int64_t>(row) * a.Hkv + hk) * kPartSplits;
    for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
        const int g = idx / HD;
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(a.part_ml + ((base + sp) * G + g) * 2));
        float L = 0.f, O = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float w = exp2f(__ldcg(a.part_ml + ((base + sp) * G + g) * 2) - M);
            L += __ldcg(a.part_ml + ((base + sp) * G + g) * 2 + 1) * w;
            O += __ldcg(a.part_o + (base + sp) * G * HD + idx) * w;
        }
        out[static_cast<int64_t>(row) * a.H * HD + (hk * G) * HD + idx] = __float2bfloat16_rn(O / L);
    }
}

template <int HD, int G>
void decode_launch(const __nv_bfloat16* q, const __nv_bfloat16* kv_layer, __nv_bfloat16* out, const DecodeAttnArgs& a,
                   int max_rows, cudaStream_t st) {
    constexpr int KB = HD <= 64 ? 32 : 16;
    constexpr int smem = 4 * (4 * KB * HD) * 2 + (8 * G + 4 * G * HD) * 4;
    static bool cfg = false;
    if (!cfg) {
        SW_CUDA(cudaFuncSetAttribute(attn_decode_kernel<HD, G, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    // grid x: the most splits any row can take at this bucket size (the kernel
    // picks <= gridDim.x per row at run time), plus what the smem page list needs
    DecodeAttnArgs args = a;
    const int want = std::max(1, std::min(a.max_splits, cdiv(a.target_ctas, max_rows * a.Hkv)));
    args.max_splits = std::max(want, cdiv(a.max_ctx, kMaxChunkPages * kPage));
    dim3 grid(args.max_splits, a.Hkv, max_rows);
    launch_k(attn_decode_kernel<HD, G, KB>, grid, dim3(128), smem, st, q, kv_layer, out, args);
}

}  // namespace

void attn_prefill(const __nv_bfloat16* q, const __nv_bfloat16* kv_layer, __nv_bfloat16* out, const PrefillAttnArgs& a,
                  int max_tiles, int hd, cudaStream_t st) {
    dim3 grid(max_tiles, a.H);
    if (hd == 64) {
        const int smem = (kQRows + 4 * kKeys) * 64 * 2;
        static bool cfg = false;
        if (!cfg) {
            SW_CUDA(cudaFuncSetAttribute(attn_prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cfg = true;
        }
        attn_prefill_kernel<64><<<grid, 128, smem, st>>>(q, kv_layer, out, a);
    } else if (hd == 128) {
        const int smem = (kQRows + 4 * kKeys) * 128 * 2;
        static bool cfg = false;
        if (!cfg) {
            SW_CUDA(cudaFuncSetAttribute(attn_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cfg = true;
        }
        attn_prefill_kernel<128><<<grid, 128, smem, st>>>(q, kv_layer, out, a);
    } else {
        throw_cuda("attn_prefill: head_dim must be 64 or 128", cudaErrorInvalidValue, __FILE__, __LINE__);
    }
    SW_LAUNCH_CHECK();
}

void attn_decode(const __nv_bfloat16* q, const __nv_bfloat16* kv_layer, __nv_bfloat16* out, const DecodeAttnArgs& a,
                 int max_rows, int hd, cudaStream_t st) {
    const int G = a.H / a.Hkv;
    if (hd == 64 && G == 4) decode_launch<64, 4>(q, kv_layer, out, a, max_rows, st);
    else if (hd == 64 && G == 2) decode_launch<64, 2>(q, kv_layer, out, a, max_rows, st);
    else if (hd == 128 && G == 4) decode_launch<128, 4>(q, kv_layer, out, a, max_rows, st);
    else throw_cuda("attn_decode: unsupported (head_dim, group)", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw

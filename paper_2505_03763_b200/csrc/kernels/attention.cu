// Attention over the paged KV cache.
//
// Prefill: causal flash attention (online softmax, fp32 statistics) for a
//   varlen batch of prompts, GQA.  One CTA = 64 query rows of one head of one
//   prompt (4 warps x 16 rows); K/V stream through smem in 64-key blocks read
//   straight from the 16-token pages just written by rope_kv (double-buffered
//   cp.async, XOR-swizzled 16 B chunks for conflict-free ldmatrix); QK^T and
//   PV on the tensor cores with mma.m16n8k16 fp16 -> fp32 (q, K/V and P are fp16).
// Decode: split-KV paged attention on the tensor cores (see below); the G =
//   H/Hkv query heads sharing a kv head are packed into one mma tile so every
//   K/V byte is read once per step.  HBM-bound by design.
#include <algorithm>
#include <cstdlib>

#include "attention.cuh"
#include "attn_decode_unit.cuh"
#include "common.cuh"

namespace sw {

namespace {

using namespace attn;

constexpr int kQRows = 64;
constexpr int kKeys = 64;

template <int HD>
__global__ void __launch_bounds__(128, HD == 64 ? 4 : 2) attn_prefill_kernel(const kv_t* __restrict__ q,
                                                           const kv_t* __restrict__ kv_layer,
                                                           __nv_bfloat16* __restrict__ out, PrefillAttnArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    kv_t* sQ = reinterpret_cast<kv_t*>(smem_raw);
    kv_t* sK = sQ + kQRows * HD;       // [2][64][HD]
    kv_t* sV = sK + 2 * kKeys * HD;    // [2][64][HD]
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
        const kv_t* src = q + (start + (ok ? q0 + r : 0)) * qstride + h * HD + c * 8;
        cp_async16(sQ + swz<HD>(r, c), src, ok);
    }
    auto load_kv = [&](int blk, int buf) {
        for (int i = tid; i < kKeys * CH; i += 128) {
            const int r = i / CH, c = i % CH;
            const int key = blk * kKeys + r;
            const bool ok = key < len;
            const int page = ok ? ptab[key / kPage] : 0;
            const kv_t* base = kv_layer + static_cast<int64_t>(page) * a.page_stride +
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
        const kv_t* K = sK + buf * kKeys * HD;
        const kv_t* V = sV + buf * kKeys * HD;
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
                mma_f16(sc[2 * np], qf[ks], b[0], b[1]);
                mma_f16(sc[2 * np + 1], qf[ks], b[2], b[3]);
            }
        }
        // mask + online softmax (log2 domain).  The max runs on raw scores
        // (scale > 0 keeps the order) and the scale folds into the exponent:
        // p = 2^(s * scale - m) is one FFMA + one MUFU.EX2 per score.
        const bool edge = (blk + 1) * kKeys > q0 || (blk + 1) * kKeys > len;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = sc[nb][e];
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
            const float m_new = fmaxf(m_run[r], mx[r] * a.scale_log2);
            const float m_use = m_new == -INFINITY ? 0.f : m_new;
            alpha[r] = fast_exp2(m_run[r] - m_use);
            m_run[r] = m_new;
            mx[r] = m_use;
        }
        float rs[2] = {0.f, 0.f};
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float p = fast_exp2(fmaf(sc[nb][e], a.scale_log2, -mx[e >> 1]));
                sc[nb][e] = p;
                rs[e >> 1] += p;
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * alpha[r] + rs[r];
        // rescale O only when some row's max moved (most blocks past the first few leave it)
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int i = 0; i < HD / 8; ++i) {
                o[i][0] *= alpha[0];
                o[i][1] *= alpha[0];
                o[i][2] *= alpha[1];
                o[i][3] *= alpha[1];
            }
        }
        // O += P V
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4];
            pa[0] = pack_h2(sc[2 * kk][0], sc[2 * kk][1]);
            pa[1] = pack_h2(sc[2 * kk][2], sc[2 * kk][3]);
            pa[2] = pack_h2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
            pa[3] = pack_h2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
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
// One CTA = one unit (row, kv head, split of the context); see attn_decode_unit.cuh.
// NS-stage per-warp K/V rings: NS = 3 keeps 2 blocks per warp in flight at two
// CTAs per SM (more bytes in flight per SM than 3 CTAs x double buffers).
// SW_ATTN_LASTWAVE_TRIGGER=0 disables the last-wave early trigger (A/B)
__device__ __constant__ bool kEarlyTrigger_c = true;
#define kEarlyTrigger kEarlyTrigger_c

template <int HD, int G, int KB, int NS>
__global__ void __launch_bounds__(128, NS == 2 ? 3 : (NS == 3 ? 2 : 1))
    attn_decode_kernel(const kv_t* __restrict__ q, const kv_t* __restrict__ kv_layer,
                       __nv_bfloat16* __restrict__ out, DecodeAttnArgs a) {
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ uint32_t s_last;
    __shared__ int32_t s_pages[kMaxChunkPages];
    // the step's metadata was copied before its first kernel: readable before the wait
    const int n_rows = a.meta->n;
    const int row = blockIdx.z;
    if (row >= n_rows) return;
    const int ctx = a.meta->pos[row] + 1;
    // splits chosen at run time: only as many as it takes to reach
    // a.target_ctas CTAs, each warp keeping >= 1 key block
    const SplitPlan plan = decode_split_plan<KB>(ctx, cdiv(a.target_ctas, n_rows * a.Hkv), static_cast<int>(gridDim.x));
    // The successor GEMM (~112 KB CTAs) may only launch once this kernel's last wave is resident
    // (earlier, its CTAs would take the slots later waves need): the CTAs of the last
    // ~target_ctas units trigger at their start, the others count as triggered when they exit.
    // Measured (tools/step_time.py): Llama-1B b=64 step 1.030 -> 1.006 ms; Llama-8B b=128 ctx 1024
    // 6.78 -> 7.17 ms (its attention streams at HBM peak and the GEMM's prefetch competes) -> hd 64 only.
    if (HD == 64 && kEarlyTrigger && row >= n_rows - cdiv(a.target_ctas, a.Hkv * max(1, plan.splits)))
        griddep_launch_dependents();
    const int split = blockIdx.x;
    if (split >= plan.splits) return;
    decode_unit<HD, G, KB, NS>(a, q, kv_layer, out, row, blockIdx.y, split, plan, ctx, dsm, s_pages, &s_last,
                               threadIdx.x, [] { __syncthreads(); }, [] { griddep_wait(); });
}

void set_early_trigger_once() {
    static bool done = [] {
        const char* v = std::getenv("SW_ATTN_LASTWAVE_TRIGGER");
        const bool on = !(v && *v && std::atoi(v) == 0);
        SW_CUDA(cudaMemcpyToSymbol(kEarlyTrigger_c, &on, sizeof(on)));
        return true;
    }();
    (void)done;
}

template <int HD, int G, int NS>
void decode_launch_ns(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out,
                      const DecodeAttnArgs& a, int max_rows, cudaStream_t st) {
    constexpr int KB = decode_kb<HD>();
    constexpr int smem = decode_unit_smem<HD, G, NS>();
    static bool cfg = false;
    if (!cfg) {
        SW_CUDA(cudaFuncSetAttribute(attn_decode_kernel<HD, G, KB, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
        cfg = true;
    }
    // grid x: the most splits any row can take at this bucket size (the kernel
    // picks <= gridDim.x per row at run time), plus what the smem page list needs
    set_early_trigger_once();
    DecodeAttnArgs args = a;
    const int want = std::max(1, std::min(a.max_splits, cdiv(a.target_ctas, max_rows * a.Hkv)));
    args.max_splits = std::max(want, cdiv(a.max_ctx, kMaxChunkPages * kPage));
    dim3 grid(args.max_splits, a.Hkv, max_rows);
    launch_k(attn_decode_kernel<HD, G, KB, NS>, grid, dim3(128), smem, st, q, kv_layer, out, args);
}

template <int HD, int G>
void decode_launch(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out, const DecodeAttnArgs& a,
                   int max_rows, cudaStream_t st) {
    static const int ns = [] {
        const char* v = std::getenv("SW_ATTN_STAGES");  // measured: 3 (profiles/r01b/step_ablation.txt)
        return v && *v ? std::atoi(v) : 3;
    }();
    if (ns == 3) decode_launch_ns<HD, G, 3>(q, kv_layer, out, a, max_rows, st);
    else if (ns == 4) decode_launch_ns<HD, G, 4>(q, kv_layer, out, a, max_rows, st);
    else decode_launch_ns<HD, G, 2>(q, kv_layer, out, a, max_rows, st);
}

}  // namespace

void attn_prefill(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out, const PrefillAttnArgs& a,
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

void attn_decode(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out, const DecodeAttnArgs& a,
                 int max_rows, int hd, cudaStream_t st) {
    const int G = a.H / a.Hkv;
    if (hd == 64 && G == 4) decode_launch<64, 4>(q, kv_layer, out, a, max_rows, st);
    else if (hd == 64 && G == 2) decode_launch<64, 2>(q, kv_layer, out, a, max_rows, st);
    else if (hd == 128 && G == 4) decode_launch<128, 4>(q, kv_layer, out, a, max_rows, st);
    else throw_cuda("attn_decode: unsupported (head_dim, group)", cudaErrorInvalidValue, __FILE__, __LINE__);
}

}  // namespace sw

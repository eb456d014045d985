// Host-facing interface of the tcgen05 GEMM (see gemm_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace sw {

enum GemmEpilogue : int {
    EPI_STORE = 0,      // bf16 out
    EPI_RESID = 1,      // fp32 out += acc (residual stream)
    EPI_SWIGLU = 2,     // [gate 64 | up 64] feature blocks -> bf16 silu(g)*u
    EPI_ARGMAX = 3,     // packed (value, index) atomicMax per token
    EPI_STORE_F32 = 4,  // fp32 out
    EPI_QKV_ROPE = 5,   // RoPE on q/k heads, q -> fp16 buffer, k/v -> paged fp16 KV cache
};

constexpr int kSsStride = 256;  // tokens per sum(x^2) partial row (max decode rows)

// Decode-only epilogue fusions (swap-AB).
struct DecodeFusion {
    // RMSNorm folded into the consumer GEMM: acc *= rsqrt(sum_p ss_parts[p][t] / norm_dim + eps),
    // partial sums of squares added in a fixed order (deterministic); B is
    // bf16(x * gain) written by the producer (x_gain below)
    const float* ss_parts = nullptr;  // [ss_nparts][kSsStride]
    int ss_nparts = 0;
    float norm_eps = 1e-5f;
    int norm_dim = 0;
    // RESID producer side: write bf16(x) for the next GEMM and this tile's
    // partial sum(x^2) per token to ss_part_out[tile][t]
    __nv_bfloat16* x_bf16 = nullptr;
    const __nv_bfloat16* x_gain = nullptr;  // the consuming RMSNorm's gain: x_bf16 = bf16(x * gain)
    float* ss_part_out = nullptr;
    // QKV_ROPE: per-token position / slot, page table, cos/sin table, outputs
    const int32_t* pos = nullptr;
    const int32_t* slot = nullptr;
    const int32_t* page_table = nullptr;
    int max_pages = 0, page_tokens = 16;
    const float2* rope_cs = nullptr;
    __half* q_out = nullptr;     // fp16 (kv_t): the attention operands
    __half* kv_layer = nullptr;
    long long page_stride = 0;
    int H = 0, Hkv = 0, hd = 0;
};

struct GemmArgs {
    int M, N, K;
    int mode;
    void* out;
    int ldo;
    int valid_tokens;
    const int* live_tokens;  // optional device bound (graph-captured decode)
    unsigned long long* argmax;
    int feature_offset;
    int stream_k;        // decode: (tile, K-block) iterations split evenly over the CTAs
    int trace;           // diagnostic: SW_DEC_TRACE=1 stamps per-CTA phase times (gemm_decode.cu)
    float* ws;           // stream-K partial tiles [ctas][2][BN][128]
    unsigned* counters;  // stream-K arrival counters [tiles], zero between launches
    DecodeFusion fx;
};

// Y[t, f] = sum_k X[t, k] W[f, k] over `tokens` rows of X and `features` rows of W.
struct GemmProblem {
    const void* X;   // bf16 [x_rows, K] (x_rows >= tokens; rows past `tokens` are ignored)
    int64_t x_rows;
    const void* W;   // bf16 [w_rows, K]
    int64_t w_rows;
    int tokens;
    const int* live_tokens;  // optional device-side live row count (<= tokens)
    int features;    // rows of W used (from row 0)
    int K;
    int mode;        // GemmEpilogue
    bool swap;       // decode: weights as the UMMA M operand
    void* out;       // STORE/SWIGLU: bf16 [tokens, ldo]; RESID: fp32 [tokens, ldo]
    int ldo;
    unsigned long long* argmax;  // ARGMAX: packed key per token
    int feature_offset;          // ARGMAX: index of W row 0 in the full vocabulary
    // optional split-K scratch (swap mode): enables split-K when present
    float* ws = nullptr;
    size_t ws_floats = 0;
    unsigned* counters = nullptr;
    int n_counters = 0;
    DecodeFusion fx;  // swap-mode epilogue fusions
    bool lean = false;  // normal mode: 128-wide tiles in ~105 KB smem (co-resident with decode CTAs)
    int yield_tiles = 0;  // normal mode: > 0 caps the tiles per CTA (grid = tiles / k): CTAs retire
                          // every ~k tiles, so higher-priority decode CTAs get SMs between them
};

// 2-D map of 16-bit rows (bf16, or fp16 for the KV arena), box 64 x box_rows, SWIZZLE_128B
CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, bool fp16 = false);
CUtensorMap make_tmap_heads(const void* base, uint64_t rows, uint64_t heads, uint64_t hd);
const CUtensorMap& tmap_cached(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
void gemm_run(const GemmProblem& p, cudaStream_t st);
// decode projections: split-K over a cluster (gemm_decode.cu)
int gemm_decode_splits(int tiles, int nk, int ctas);
size_t gemm_decode_ws_floats(int tiles, int S, int bn);
void gemm_decode_run(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int bn, int S, int tiles,
                     cudaStream_t st);
// decode projections, stream-K over a persistent grid of P CTAs (gemm_decode2.cu)
size_t gemm_decode_sk_ws_floats(int P, int bn);
void gemm_decode_sk_run(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args, int bn, int tiles, int P,
                        cudaStream_t st);

}  // namespace sw

// Model + KV arena objects behind the kernel-level C-ABI (sw_model / sw_kv).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <tuple>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/splitwise.h"
#include "../kernels/attention.cuh"
#include "../kernels/elementwise.cuh"

namespace sw {

struct LayerWeights {
    __nv_bfloat16* wqkv;  // [(H + 2Hkv) hd, d]  rows: q heads | k heads | v heads
    __nv_bfloat16* wo;    // [d, H hd]
    __nv_bfloat16* wgu;   // [2 ffn, d]  blocks of 128 rows: [gate 64 | up 64]
    __nv_bfloat16* wd;    // [d, ffn]
    __nv_bfloat16* g_attn;
    __nv_bfloat16* g_mlp;
};

// Per-phase activation workspace (one per stream: prefill and decode never
// share buffers, so the two phases can run concurrently).
struct Workspace {
    int rows = 0;
    float* x = nullptr;              // [rows, d] residual stream, fp32
    __nv_bfloat16* xn = nullptr;     // [rows, d]
    float* qkv = nullptr;            // [rows, (H + 2Hkv) hd] fp32 (rounded once, after RoPE)
    kv_t* q = nullptr;               // [rows, H hd] roped, fp16
    __nv_bfloat16* attn = nullptr;   // [rows, H hd]
    __nv_bfloat16* act = nullptr;    // [rows, ffn]
    __nv_bfloat16* xlast = nullptr;  // [256, d] rows feeding the LM head
    unsigned long long* keys = nullptr;  // [256] packed argmax
    // decode only
    StepMeta* meta = nullptr;
    float* ss = nullptr;  // [2][kMaxDecodeRows] sum(x^2) accumulators for the folded RMSNorms
    float* splitk_ws = nullptr;  // split-K partial tiles of the decode GEMMs
    size_t splitk_floats = 0;
    unsigned* splitk_cnt = nullptr;
    float* part_o = nullptr;
    float* part_ml = nullptr;
    unsigned* attn_cnt = nullptr;  // split-KV arrival counters [rows][Hkv]
    // flat decode attention: per-warp partials
    float* flat_o = nullptr;
    float* flat_ml = nullptr;
    // prefill only: device metadata block
    int32_t* pmeta = nullptr;
    size_t pmeta_bytes = 0;
};

struct PinnedRing {
    std::vector<void*> slots;
    std::vector<cudaEvent_t> done;
    size_t bytes = 0;
    int next = 0;
};

struct DecodeGraph {
    cudaGraphExec_t exec = nullptr;
    int eager_runs = 0;
    unsigned long long kernels = 0;  // kernel nodes in the graph
};

}  // namespace sw

struct sw_model {
    sw_model_desc desc{};
    int device = 0;
    void* weight_arena = nullptr;
    size_t weight_bytes = 0;
    __nv_bfloat16* emb = nullptr;
    __nv_bfloat16* lm = nullptr;
    __nv_bfloat16* g_final = nullptr;
    std::vector<sw::LayerWeights> layers;
    std::map<std::string, std::pair<void*, int64_t>> tensors;
    float* inv_freq = nullptr;
    float2* rope_cs = nullptr;  // [kMaxPositions][hd/2] (cos, sin)
    sw::Workspace pre;
    sw::Workspace mix;  // decode-row scratch of fused mixed steps (StepMeta, split-KV partials); lazy
    // decode lanes: one workspace + staging ring + graph set per concurrent
    // decode stream (lanes of different instances may step at the same time)
    static constexpr int kMaxDecodeLanes = 4;
    sw::Workspace dec[kMaxDecodeLanes];
    sw::PinnedRing pre_ring, mix_ring, dec_ring[kMaxDecodeLanes];
    // (arena, row bucket, lane | mode, partition): a graph runs in the context it was captured in
    std::map<std::tuple<const sw_kv*, int, int, const void*>, sw::DecodeGraph> graphs;
    unsigned long long* scratch_u64 = nullptr;
};

struct sw_kv {
    sw_model* model = nullptr;
    int64_t n_pages = 0;
    int32_t n_slots = 0, max_pages = 0, max_out = 0;
    int page_tokens = 16;
    sw::kv_t* pages = nullptr;       // [L][n_pages][2][Hkv][B][hd] fp16
    int32_t* page_table = nullptr;   // [n_slots][max_pages]
    int32_t* last_token = nullptr;   // [n_slots]
    int32_t* out_tokens = nullptr;   // [n_slots][max_out]
    int64_t layer_stride = 0;        // elements per layer
    int64_t page_stride = 0;         // elements per page (one layer)
    int chunk = 256;
    int max_splits = 1;
    // the whole arena as one 2-D TMA map of head_dim-element rows (flat decode attention)
    CUtensorMap tm_kv{};
    bool tm_kv_ok = false;
};

namespace sw {
constexpr int kMaxPositions = 32768;  // RoPE table extent (max context)
// Forward passes (stream-ordered; host arrays staged internally).
// lean: 128-wide prefill GEMM tiles in ~105 KB smem, so decode CTAs can share the SMs
// yield_tiles: > 0 caps the tiles per GEMM CTA (decode CTAs interleave at tile granularity)
void prefill_forward(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st, bool lean = false,
                     int yield_tiles = 0);
// One fused mixed step (the split-phase co-execution of a prompt chunk and a
// token step): the decode rows of `dec` (sw_decode_enqueue semantics) ride in
// the prefill pass of `pre` -- every projection GEMM runs once over
// [prompt tokens | decode rows] (the weights stream once for both phases),
// the prompts attend causally with the tcgen05 prefill kernel, the decode rows
// over their paged contexts with the decode kernel.  All prompts and decode
// rows must fit one launch (tokens + rows <= max_prefill_tokens, prompts + rows
// <= 256).  logits (optional, parity) = prompts' last positions, then decode rows.
void mixed_forward(sw_model* m, sw_kv* kv, const sw_batch& pre, const sw_batch& dec, cudaStream_t st,
                   float* logits_out = nullptr);
void decode_forward(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st, bool use_graph, int lane = 0,
                    int lanes = 1);
int decode_bucket(int n);
}  // namespace sw

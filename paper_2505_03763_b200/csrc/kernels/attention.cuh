// Host-facing interface of the attention kernels (attention.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "elementwise.cuh"

namespace sw {

// Prefill: 64-row query tiles over a varlen batch (host-built tile list).
struct PrefillAttnArgs {
    const int* n_tiles;        // device
    const int32_t* tile_seq;   // device [tiles]
    const int32_t* tile_q0;    // device [tiles]
    const int32_t* cu_seqlens; // device [seqs + 1]
    const int32_t* seq_slot;   // device [seqs]
    const int32_t* page_table; // device [slots][max_pages]
    int max_pages;
    int page_tokens;
    int64_t page_stride;  // elements per page (one layer)
    int64_t kv_stride;    // elements from K to V inside a page
    int H, Hkv;
    float scale_log2;     // log2(e) / sqrt(head_dim)
};

struct DecodeAttnArgs {
    const StepMeta* meta;
    const int32_t* page_table;
    int max_pages;
    int page_tokens;
    int64_t page_stride;
    int64_t kv_stride;
    int H, Hkv;
    float scale_log2;
    int chunk;       // keys per split
    int max_splits;  // grid x; splits past the context exit
    float* part_o;   // [rows][Hkv][max_splits][G][hd]
    float* part_ml;  // [rows][Hkv][max_splits][G][2]
    unsigned* counters;  // [rows][Hkv] split arrivals, zero between launches
    int target_ctas;     // split-KV: split until rows * Hkv * splits reaches this
    int max_ctx;         // longest context the arena holds (sizes the grid)
};

// Prefill on tcgen05 (attn_prefill_tc.cu): 128-row query tiles (host-built
// list), Q through a 3-D TMA map over [tokens][H][hd], K/V through the arena map.
struct PrefillTcArgs {
    const int* n_tiles;        // device
    const int32_t* tile_seq;   // device [tiles]
    const int32_t* tile_q0;    // device [tiles]
    const int32_t* cu_seqlens; // device [seqs + 1]
    const int32_t* seq_pos0;   // device [seqs]: first position of each prompt chunk (multiple of 128), or null
    const int32_t* seq_slot;   // device [seqs]
    const int32_t* page_table; // device [slots][max_pages]
    int max_pages;
    int H, Hkv;
    float scale_log2;
    int layer_row0;  // arena-map row of (layer, page 0, K, head 0)
    int page_rows;   // arena-map rows per page
    int v_rows;      // K -> V rows inside a page
};
// persistent: one CTA per SM looping over (tile, head pair) items -- amortises the CTA
// prologue for short prompts; long prompts (uneven causal items) keep one item per CTA
void attn_prefill_tc(const CUtensorMap& tm_q, const CUtensorMap& tm_kv, __nv_bfloat16* out, const PrefillTcArgs& a,
                     int max_tiles, int hd, bool persistent, cudaStream_t st);

// Flat page-balanced decode attention (attn_decode_flat.cu): persistent grid,
// TMA page-slice loads through a 2-D map of the whole KV arena (rows of hd
// elements; K slice of (layer l, page p, kv head h) at row
// layer_row0 + p * page_rows + h * 16, its V slice v_rows further).
struct DecodeFlatArgs {
    const StepMeta* meta;
    const int32_t* page_table;
    int max_pages;
    int H, Hkv;
    float scale_log2;
    int layer_row0;
    int page_rows;
    int v_rows;
    float* part_o;       // [2 * warps][G][hd]
    float* part_ml;      // [2 * warps][G][2]
    unsigned* counters;  // [rows][Hkv], zero between launches
};
// partial slots (each G x hd floats) the flat kernel needs on `sms` SMs
size_t attn_decode_flat_part_rows(int sms);

void attn_prefill(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out, const PrefillAttnArgs& a,
                  int max_tiles, int hd, cudaStream_t st);
void attn_decode(const kv_t* q, const kv_t* kv_layer, __nv_bfloat16* out, const DecodeAttnArgs& a,
                 int max_rows, int hd, cudaStream_t st);
void attn_decode_flat(const CUtensorMap& tm_kv, const kv_t* q, __nv_bfloat16* out, const DecodeFlatArgs& a,
                      int ctas, int hd, int G, cudaStream_t st);

}  // namespace sw

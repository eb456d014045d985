// Declarations of the HBM-bound helper kernels (elementwise.cu) and the
// per-launch metadata blocks the host stages with one H2D copy.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sw {

// storage type of roped q and the paged K/V cache (see common.cuh)
using kv_t = __half;

constexpr int kMaxDecodeRows = 256;

// Decode step metadata, device resident; the host fills a pinned copy and
// issues one cudaMemcpyAsync per step.  Kernels read `n` at run time, so a
// CUDA graph captured for a row bucket serves every batch up to its size.
struct StepMeta {
    int32_t n;
    int32_t pad_[31];
    int32_t slot[kMaxDecodeRows];
    int32_t pos[kMaxDecodeRows];       // position of the fed token (= context - 1)
    int32_t token[kMaxDecodeRows];     // -1: slot's last generated token
    int32_t new_page[kMaxDecodeRows];  // -1: none; else page for index pos / B
    int32_t out_index[kMaxDecodeRows];
};

void init_tensor(__nv_bfloat16* dst, int64_t rows, int cols, uint64_t seed, int k, int fan_in, int blk, int blk_stride,
                 int blk_off, cudaStream_t st);
void fill_bf16(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t st);
void checksum_bf16(const void* p, int64_t n, unsigned long long* out_dev, cudaStream_t st);

void embed(const StepMeta* meta, int max_rows, const __nv_bfloat16* emb, const __nv_bfloat16* gain, float* x,
           __nv_bfloat16* xb, float* ss_a, int d, const int32_t* last_token, int32_t* page_table, int max_pages,
           int page_tokens, cudaStream_t st);
void embed_tokens(const int32_t* tokens, const int* n_tokens_dev, int rows, const __nv_bfloat16* emb, float* x, int d,
                  cudaStream_t st);
void rmsnorm(const float* x, const __nv_bfloat16* g, __nv_bfloat16* y, int rows, int d, float eps, const int* rows_dev,
             const int32_t* row_index, cudaStream_t st);
void rope_table(const float* inv_freq, float2* table, int max_pos, int half, cudaStream_t st);
void rope_kv(const float* qkv, kv_t* q_out, kv_t* kv_layer, const int32_t* tok_pos,
             const int32_t* tok_slot, const int32_t* page_table, const float2* cs_table, int rows, const int* rows_dev,
             int H, int Hkv, int hd, int max_pages, int page_tokens, cudaStream_t st);
void finalize_tokens(unsigned long long* keys, const int32_t* slot, const int32_t* out_index, int rows,
                     const int* rows_dev, int32_t* last_token, int32_t* out_tokens, int max_out, cudaStream_t st);

}  // namespace sw

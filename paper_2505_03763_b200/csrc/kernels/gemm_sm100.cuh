// Host-facing interface of the tcgen05 GEMM (see gemm_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sw {

enum GemmEpilogue : int { EPI_STORE = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_ARGMAX = 3, EPI_STORE_F32 = 4 };

struct GemmArgs {
    int M, N, K;
    int mode;
    void* out;
    int ldo;
    int valid_tokens;
    const int* live_tokens;  // optional device bound (graph-captured decode)
    unsigned long long* argmax;
    int feature_offset;
    int splits;          // split-K factor (grid z)
    float* ws;           // split-K partial tiles [tiles][splits][BN][128]
    unsigned* counters;  // split-K arrival counters [tiles], zero between launches
    int stagger;         // rotate each tile's K-block order (DRAM channel spread)
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
};

CUtensorMap make_tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
const CUtensorMap& tmap_cached(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
void gemm_run(const GemmProblem& p, cudaStream_t st);

}  // namespace sw

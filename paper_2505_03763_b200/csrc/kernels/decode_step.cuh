// Host-facing interface of the persistent decode-step kernel (decode_step.cu):
// a whole decode step -- every layer's QKV / attention / Wo / gate-up / down
// projections and the LM head -- in ONE launch of one CTA per SM.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "attention.cuh"
#include "elementwise.cuh"
#include "gemm_sm100.cuh"

namespace sw {

enum StepPhaseKind : int { PHASE_GEMM = 0, PHASE_ATTN = 1 };

// One phase of the step.  Phases run in list order; phase p+1 may only
// consume what phase p wrote after every CTA has arrived on bar[p].
struct StepPhase {
    int kind;          // StepPhaseKind
    int mode;          // GEMM: GemmEpilogue (QKV_ROPE, RESID, SWIGLU, ARGMAX)
    int w_map, x_map;  // GEMM: tensor maps of the weights [M, K] and activations [rows, K]
    int M, K;          // GEMM: weight rows (multiple of 128), reduction length (multiple of 64)
    int cnt_off;       // GEMM: this phase's split-K tile counters (StepArgs::counters + cnt_off)
    GemmArgs g;        // GEMM: epilogue arguments (out, ldo, argmax, feature_offset, fx, tokens)
    const __nv_bfloat16* q;   // ATTN: roped queries [rows, H hd]
    const __nv_bfloat16* kv;  // ATTN: this layer's paged KV cache
    __nv_bfloat16* out;       // ATTN: [rows, H hd]
};

struct StepArgs {
    const StepPhase* phases;  // device [n_phases]
    int n_phases;
    const CUtensorMap* maps;  // device, 64 B aligned
    unsigned* bar;            // device [n_phases] arrivals, zeroed before the launch
    float* ws;                // stream-K partial tiles [ctas][2][BN * 128]
    unsigned* counters;       // split-K tile counters, one block per phase, zeroed before the launch
    const StepMeta* meta;
    DecodeAttnArgs attn;      // attention arguments shared by every layer
    int attn_target;          // attention units per phase to aim for (split-KV)
    int debug_single_reducer;   // 1: the tile's first contributor reduces every column group
    unsigned long long* trace;  // optional [n_phases][ctas][8] globaltimer stamps (tools/step_trace.py)
};

bool decode_step_supported(int bn, int hd, int group);
int decode_step_stages(int bn, int hd, int group);
void decode_step_launch(const StepArgs& a, int bn, int hd, int group, int ctas, cudaStream_t st);

}  // namespace sw

// Swap-AB (decode) GEMM epilogue of the persistent kernel (gemm_sm100.cu: the
// LM head with greedy argmax) and the persistent decode-step kernel.
// Thread = output feature row of a 128-row weight tile (TMEM lane order:
// row = 32 * (warp % 4) + lane over the 4 epilogue warps); columns = tokens.
#pragma once

#include "common.cuh"
#include "gemm_sm100.cuh"

namespace sw {

// silu(g) * u; the fast reciprocal maps 1 + e^-g = inf to 0 (no IEEE slow path)
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

struct SwapEpi {
    const GemmArgs* args;
    float* xchg;            // [128][33] smem exchange
    const float* tok_inv;   // [256] smem 1/rms per token
    const int* tok_pos;     // [256] smem position per token (QKV_ROPE)
    const long long* tok_kv;  // [256] smem KV page offset per token (QKV_ROPE)
    int row, lane, quarter, n_live;
    unsigned long long* best = nullptr;  // ARGMAX: smem running max per token (flushed once per CTA)
};

// 32 fp32 values per lane -> lane j holds the warp sum of value j (31 shuffles)
__device__ __forceinline__ void transpose_sum(float (&v)[32], int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = upper ? v[i] : v[i + off];
            const float keep = upper ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
}

// 32 packed keys per lane -> lane j holds the warp max of key j (31 shuffles)
__device__ __forceinline__ void transpose_max(unsigned long long (&v)[32], int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const unsigned long long send = upper ? v[i] : v[i + off];
            const unsigned long long keep = upper ? v[i + off] : v[i];
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, send, off);
            v[i] = other > keep ? other : keep;
        }
    }
}

// Apply the fused epilogue MODE to token columns [c, c + min(32, width)) of
// feature tile m0 (vin[j] = column c + j).  Uses named barrier 1 over the 128
// epilogue threads.
template <int MODE>
__device__ __forceinline__ void emit_swap(const SwapEpi& E, int m0, int c, const float (&vin)[32], int width = 32) {
    const GemmArgs& args = *E.args;
    const DecodeFusion& fx = args.fx;
    float* xchg = E.xchg;
    const int row = E.row, lane = E.lane, quarter = E.quarter, n_live = E.n_live;
    const float* tok_inv = E.tok_inv;
    const int* tok_pos = E.tok_pos;
    const long long* tok_kv = E.tok_kv;

        const int f = m0 + row;
        const int tcount = min(min(32, width), n_live - c);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = vin[j];
        if (fx.ss_parts && MODE != EPI_RESID) {  // RMSNorm of the input rows, folded in
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < tcount) v[j] *= tok_inv[c + j];
        }
        if constexpr (MODE == EPI_STORE) {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                static_cast<__nv_bfloat16*>(args.out)[static_cast<size_t>(c + j) * args.ldo + f] =
                    __float2bfloat16_rn(v[j]);
        } else if constexpr (MODE == EPI_STORE_F32) {
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                static_cast<float*>(args.out)[static_cast<size_t>(c + j) * args.ldo + f] = v[j];
        } else if constexpr (MODE == EPI_RESID) {
            float* col = static_cast<float*>(args.out) + static_cast<size_t>(c) * args.ldo + f;
            float x[32];
            _Pragma("unroll") for (int j = 0; j < 32; ++j) x[j] =
                j < tcount ? __ldcg(col + static_cast<size_t>(j) * args.ldo) : 0.f;
            _Pragma("unroll") for (int j = 0; j < 32; ++j) {
                x[j] += v[j];
                if (j < tcount) {
                    col[static_cast<size_t>(j) * args.ldo] = x[j];
                    if (fx.x_bf16)
                        fx.x_bf16[static_cast<size_t>(c + j) * args.ldo + f] =
                            __float2bfloat16_rn(x[j] * __bfloat162float(fx.x_gain[f]));
                }
                x[j] = j < tcount ? x[j] * x[j] : 0.f;
            }
            if (fx.ss_part_out) {  // this tile's sum(x^2) per token, for the next RMSNorm
                transpose_sum(x, lane);  // lane j: the warp's partial for token c + j
                xchg[quarter * 32 + lane] = x[0];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (quarter == 0 && lane < tcount)  // fixed order over the 4 warps: deterministic
                    fx.ss_part_out[static_cast<size_t>(m0 / 128) * kSsStride + c + lane] =
                        (xchg[lane] + xchg[32 + lane]) + (xchg[64 + lane] + xchg[96 + lane]);
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
        } else if constexpr (MODE == EPI_SWIGLU) {
            // lanes 0-63 of the tile hold gate rows, 64-127 the matching up rows
            if (row >= 64) {
#pragma unroll
                for (int j = 0; j < 32; ++j) xchg[(row - 64) * 33 + j] = v[j];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (row < 64) {
                const int gi = m0 / 2 + row;
                _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount)
                    static_cast<__nv_bfloat16*>(args.out)[static_cast<size_t>(c + j) * args.ldo + gi] =
                        __float2bfloat16_rn(silu_mul(v[j], xchg[row * 33 + j]));
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        } else if constexpr (MODE == EPI_ARGMAX) {
            if (E.best) {  // per-CTA running max in smem: one global atomic per token per CTA
                unsigned long long k[32];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    k[j] = j < tcount ? argmax_key(v[j], static_cast<uint32_t>(args.feature_offset + f)) : 0ull;
                transpose_max(k, lane);
                if (lane < tcount) atomicMax(E.best + c + lane, k[0]);
                return;
            }
            _Pragma("unroll") for (int j = 0; j < 32; ++j) if (j < tcount) {
                unsigned long long key = argmax_key(v[j], static_cast<uint32_t>(args.feature_offset + f));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
                    key = other > key ? other : key;
                }
                if (lane == 0) atomicMax(args.argmax + c + j, key);
            }
        } else if constexpr (MODE == EPI_QKV_ROPE) {
            // rotate-half RoPE: row r pairs with r ^ (hd/2) inside its head
            const int hd = fx.hd, half = hd >> 1;
            const int head = f / hd, i = f % hd;
#pragma unroll
            for (int j = 0; j < 32; ++j) xchg[row * 33 + j] = v[j];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int prow = row ^ half;
            const bool is_v = head >= fx.H + fx.Hkv;
            _Pragma("unroll") for (int j = 0; j < 32; ++j) {
                if (j >= tcount) continue;
                const int t = c + j;
                const int pos = tok_pos[t];
                float out = v[j];
                if (!is_v) {
                    const float2 cs = fx.rope_cs[static_cast<int64_t>(pos) * half + (i & (half - 1))];
                    const float b = xchg[prow * 33 + j];
                    out = i < half ? v[j] * cs.x - b * cs.y : v[j] * cs.x + b * cs.y;
                }
                if (head < fx.H) {
                    fx.q_out[static_cast<size_t>(t) * fx.H * hd + f] = __float2half_rn(out);
                } else {
                    const int kvh = is_v ? head - fx.H - fx.Hkv : head - fx.H;
                    kv_t* dst = fx.kv_layer + tok_kv[t] + (is_v ? fx.page_stride / 2 : 0) +
                                         static_cast<int64_t>(kvh) * fx.page_tokens * hd + i;
                    *dst = __float2half_rn(out);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
}

}  // namespace sw

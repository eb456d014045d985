// Fused per-token epilogue of the decode projection GEMMs (gemm_decode.cu,
// gemm_decode2.cu): one warp per token, 4 features per lane, so every global
// access is a 16 B (fp32) or 8 B (bf16) vector.
#pragma once

#include "common.cuh"
#include "gemm_epilogue.cuh"
#include "gemm_sm100.cuh"

namespace sw {
namespace dec_epi {

// Per-token epilogue context (shared memory tables filled once per CTA).
struct TokCtx {
    const GemmArgs* a;
    const float* tok_inv;      // 1/rms of each input row (folded RMSNorm)
    const int* tok_pos;        // QKV_ROPE: position of each row
    const long long* tok_kv;   // QKV_ROPE: KV-cache element offset of each row's slot
    int m0;                    // first weight row (output feature) of the tile
};

// Fused epilogue for token t over tile features [4*lane, 4*lane + 4): one warp
// per token, so every global access is a 16 B (fp32) or 8 B (bf16) vector and
// a warp covers the tile's 128 features of the token contiguously.  Pairs of
// features that meet in an epilogue (SwiGLU gate/up, RoPE rotate-half
// partners) are lanes apart and exchanged by shuffles.  t is warp uniform.
// Global inputs of emit_tok that do not depend on the accumulator (residual
// row, RoPE cos/sin), loaded one token ahead so their latency overlaps the
// previous token's epilogue.
struct TokPre {
    float4 a, b;
};

template <int MODE>
__device__ __forceinline__ TokPre pre_tok(const TokCtx& c, int t, int lane) {
    const GemmArgs& args = *c.a;
    const int f0 = c.m0 + 4 * lane;
    TokPre p{};
    if constexpr (MODE == EPI_RESID) {
        p.a = __ldcg(reinterpret_cast<const float4*>(static_cast<const float*>(args.out) +
                                                     static_cast<size_t>(t) * args.ldo + f0));
    } else if constexpr (MODE == EPI_QKV_ROPE) {
        const DecodeFusion& fx = args.fx;
        const int hd = fx.hd, half = hd >> 1;
        const int head = f0 / hd, d0 = f0 - head * hd;
        if (head < fx.H + fx.Hkv) {
            const float4* cs4 = reinterpret_cast<const float4*>(fx.rope_cs + static_cast<int64_t>(c.tok_pos[t]) * half +
                                                                (d0 & (half - 1)));
            p.a = __ldg(cs4);
            p.b = __ldg(cs4 + 1);
        }
    }
    return p;
}

template <int MODE>
__device__ __forceinline__ void emit_tok(const TokCtx& c, int t, int lane, float4 v, const TokPre& pre) {
    const GemmArgs& args = *c.a;
    const DecodeFusion& fx = args.fx;
    const int i0 = 4 * lane;
    const int f0 = c.m0 + i0;
    if (fx.ss_parts && MODE != EPI_RESID) {  // RMSNorm of the input row, folded in
        const float s = c.tok_inv[t];
        v.x *= s;
        v.y *= s;
        v.z *= s;
        v.w *= s;
    }
    if constexpr (MODE == EPI_STORE) {
        *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.out) + static_cast<size_t>(t) * args.ldo + f0) =
            make_uint2(pack_bf2(v.x, v.y), pack_bf2(v.z, v.w));
    } else if constexpr (MODE == EPI_STORE_F32) {
        *reinterpret_cast<float4*>(static_cast<float*>(args.out) + static_cast<size_t>(t) * args.ldo + f0) = v;
    } else if constexpr (MODE == EPI_RESID) {
        float4* px = reinterpret_cast<float4*>(static_cast<float*>(args.out) + static_cast<size_t>(t) * args.ldo + f0);
        float4 x = pre.a;
        x.x += v.x;
        x.y += v.y;
        x.z += v.z;
        x.w += v.w;
        *px = x;
        if (fx.x_bf16) {  // the next GEMM's B operand: bf16(x * g) of the consuming RMSNorm
            const uint2 g = __ldg(reinterpret_cast<const uint2*>(fx.x_gain + f0));
            *reinterpret_cast<uint2*>(fx.x_bf16 + static_cast<size_t>(t) * args.ldo + f0) =
                make_uint2(pack_bf2(x.x * bf_lo(g.x), x.y * bf_hi(g.x)), pack_bf2(x.z * bf_lo(g.y), x.w * bf_hi(g.y)));
        }
        if (fx.ss_part_out) {  // this tile's sum(x^2) of the token, for the next RMSNorm (fixed tree)
            const float ss = warp_sum((x.x * x.x + x.y * x.y) + (x.z * x.z + x.w * x.w));
            if (lane == 0) fx.ss_part_out[static_cast<size_t>(c.m0 / 128) * kSsStride + t] = ss;
        }
    } else if constexpr (MODE == EPI_SWIGLU) {
        // tile rows [gate 64 | up 64]: lane l (< 16) holds gate features, lane l + 16 the matching up features
        float4 u;
        u.x = __shfl_xor_sync(0xffffffffu, v.x, 16);
        u.y = __shfl_xor_sync(0xffffffffu, v.y, 16);
        u.z = __shfl_xor_sync(0xffffffffu, v.z, 16);
        u.w = __shfl_xor_sync(0xffffffffu, v.w, 16);
        if (lane < 16)
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.out) + static_cast<size_t>(t) * args.ldo +
                                      c.m0 / 2 + i0) =
                make_uint2(pack_bf2(silu_mul(v.x, u.x), silu_mul(v.y, u.y)),
                           pack_bf2(silu_mul(v.z, u.z), silu_mul(v.w, u.w)));
    } else if constexpr (MODE == EPI_QKV_ROPE) {
        // rotate-half RoPE inside each head: feature d pairs with d ^ (hd/2), i.e. lane ^ (hd/8)
        const int hd = fx.hd, half = hd >> 1;
        const int head = f0 / hd, d0 = f0 - head * hd;
        float4 p;
        p.x = __shfl_xor_sync(0xffffffffu, v.x, half / 4);
        p.y = __shfl_xor_sync(0xffffffffu, v.y, half / 4);
        p.z = __shfl_xor_sync(0xffffffffu, v.z, half / 4);
        p.w = __shfl_xor_sync(0xffffffffu, v.w, half / 4);
        const bool is_v = head >= fx.H + fx.Hkv;
        float4 o = v;
        if (!is_v) {
            const float4 ca = pre.a, cb = pre.b;  // (cos, sin) of d0, d0+1 | d0+2, d0+3
            const float sg = d0 < half ? -1.f : 1.f;
            o.x = v.x * ca.x + sg * p.x * ca.y;
            o.y = v.y * ca.z + sg * p.y * ca.w;
            o.z = v.z * cb.x + sg * p.z * cb.y;
            o.w = v.w * cb.z + sg * p.w * cb.w;
        }
        const uint2 packed = make_uint2(pack_h2(o.x, o.y), pack_h2(o.z, o.w));
        if (head < fx.H) {
            *reinterpret_cast<uint2*>(fx.q_out + static_cast<size_t>(t) * fx.H * hd + f0) = packed;
        } else {
            const int kvh = is_v ? head - fx.H - fx.Hkv : head - fx.H;
            *reinterpret_cast<uint2*>(fx.kv_layer + c.tok_kv[t] + (is_v ? fx.page_stride / 2 : 0) +
                                      static_cast<int64_t>(kvh) * fx.page_tokens * hd + d0) = packed;
        }
    }
}


// Per-token tables every epilogue needs, filled once per CTA by `nthreads`
// threads starting at thread index e: 1/rms of each input row (folded RMSNorm)
// and, for QKV_ROPE, each row's position and KV-cache element offset.
template <int MODE>
__device__ __forceinline__ void fill_tok_tables(const GemmArgs& args, int n_live, int e, int nthreads, float* tok_inv,
                                                int* tok_pos, long long* tok_kv) {
    const DecodeFusion& fx = args.fx;
    for (int t = e; t < n_live; t += nthreads) {
        if (fx.ss_parts) {
            float ss = 0.f;
            for (int q0 = 0; q0 < fx.ss_nparts; q0 += 16) {
                float p[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    p[q] = q0 + q < fx.ss_nparts ? __ldcg(fx.ss_parts + (q0 + q) * kSsStride + t) : 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q) ss += p[q];  // fixed order: deterministic
            }
            tok_inv[t] = rsqrtf(ss / static_cast<float>(fx.norm_dim) + fx.norm_eps);
        }
        if constexpr (MODE == EPI_QKV_ROPE) {
            const int pos = fx.pos[t];
            const int page = fx.page_table[static_cast<int64_t>(fx.slot[t]) * fx.max_pages + pos / fx.page_tokens];
            tok_pos[t] = pos;
            tok_kv[t] = static_cast<long long>(page) * fx.page_stride + static_cast<long long>(pos % fx.page_tokens) * fx.hd;
        }
    }
}

}  // namespace dec_epi
}  // namespace sw

// HBM-bound helper kernels of both phases: synthetic weight init, embedding
// gather (+ page-table install for decode), RMSNorm, RoPE + paged-KV scatter,
// and the greedy-token finalize that follows the LM-head argmax GEMM.
#include <algorithm>

#include "common.cuh"
#include "elementwise.cuh"

namespace sw {

// ---------------------------------------------------------------- weights
// dst row for logical row r: (r / blk) * blk_stride + blk_off + r % blk.
__global__ void init_tensor_kernel(__nv_bfloat16* __restrict__ dst, int64_t rows, int cols, uint64_t tseed,
                                   double scale, int blk, int blk_stride, int blk_off) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = smx_mix(tseed + static_cast<uint64_t>(i + 1) * 0x9e3779b97f4a7c15ULL);
        const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
        const float w = __double2float_rn((2.0 * u - 1.0) * scale);
        const int64_t r = i / cols, c = i % cols;
        const int64_t dr = (r / blk) * blk_stride + blk_off + r % blk;
        dst[dr * cols + c] = __float2bfloat16_rn(w);
    }
}

void init_tensor(__nv_bfloat16* dst, int64_t rows, int cols, uint64_t seed, int k, int fan_in, int blk,
                 int blk_stride, int blk_off, cudaStream_t st) {
    const uint64_t tseed = seed ^ (static_cast<uint64_t>(k) * 0x9e3779b97f4a7c15ULL);
    const double scale = sqrt(3.0 / static_cast<double>(fan_in));
    init_tensor_kernel<<<148 * 16, 256, 0, st>>>(dst, rows, cols, tseed, scale, blk <= 0 ? (int)rows : blk,
                                                 blk <= 0 ? (int)rows : blk_stride, blk_off);
    SW_LAUNCH_CHECK();
}

__global__ void fill_bf16_kernel(__nv_bfloat16* dst, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(v);
}
void fill_bf16(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t st) {
    fill_bf16_kernel<<<148, 256, 0, st>>>(dst, n, v);
    SW_LAUNCH_CHECK();
}

// FNV-style order-dependent checksum of a bf16 buffer (weight parity tests).
__global__ void checksum_kernel(const uint16_t* __restrict__ p, int64_t n, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += smx_mix(static_cast<uint64_t>(p[i]) ^ (static_cast<uint64_t>(i) << 16));
    atomicAdd(out, acc);
}
void checksum_bf16(const void* p, int64_t n, unsigned long long* out_dev, cudaStream_t st) {
    checksum_kernel<<<148 * 4, 256, 0, st>>>(static_cast<const uint16_t*>(p), n, out_dev);
    SW_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- embedding
// Decode step head, one CTA per row: install the step's new page, gather the
// embedding of the fed token (the slot's device-resident last token unless
// explicit tokens are given) and emit what the first fused GEMM consumes:
// x (fp32 residual), bf16(x * g) (its B operand, g = layer 0's attention-norm
// gain) and sum(x^2) (its RMSNorm scale, as a single partial row).
__global__ void embed_kernel(const StepMeta* __restrict__ meta, const __nv_bfloat16* __restrict__ emb,
                             const __nv_bfloat16* __restrict__ gain, float* __restrict__ x,
                             __nv_bfloat16* __restrict__ xb, float* __restrict__ ss_a,
                             int d, const int32_t* __restrict__ last_token,
                             int32_t* __restrict__ page_table, int max_pages, int page_tokens) {
    griddep_launch_dependents();
    griddep_wait();
    const int row = blockIdx.x;
    if (row >= meta->n) return;
    const int slot = meta->slot[row];
    int tok = meta->token[row];
    if (tok < 0) tok = last_token[slot];
    if (threadIdx.x == 0 && meta->new_page[row] >= 0)
        page_table[static_cast<int64_t>(slot) * max_pages + meta->pos[row] / page_tokens] = meta->new_page[row];
    const uint4* src = reinterpret_cast<const uint4*>(emb + static_cast<int64_t>(tok) * d);
    float4* dst = reinterpret_cast<float4*>(x + static_cast<int64_t>(row) * d);
    uint4* dstb = reinterpret_cast<uint4*>(xb + static_cast<int64_t>(row) * d);
    const uint4* g4 = reinterpret_cast<const uint4*>(gain);
    float ss = 0.f;
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
        const uint4 v = src[i];
        const float4 a = make_float4(bf_lo(v.x), bf_hi(v.x), bf_lo(v.y), bf_hi(v.y));
        const float4 b = make_float4(bf_lo(v.z), bf_hi(v.z), bf_lo(v.w), bf_hi(v.w));
        dst[2 * i] = a;
        dst[2 * i + 1] = b;
        const uint4 g = __ldg(g4 + i);
        dstb[i] = make_uint4(pack_bf2(a.x * bf_lo(g.x), a.y * bf_hi(g.x)), pack_bf2(a.z * bf_lo(g.y), a.w * bf_hi(g.y)),
                             pack_bf2(b.x * bf_lo(g.z), b.y * bf_hi(g.z)), pack_bf2(b.z * bf_lo(g.w), b.w * bf_hi(g.w)));
        ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
    }
    __shared__ float red[32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        ss_a[row] = t;
    }
}

void embed(const StepMeta* meta, int max_rows, const __nv_bfloat16* emb, const __nv_bfloat16* gain, float* x,
           __nv_bfloat16* xb, float* ss_a, int d, const int32_t* last_token, int32_t* page_table, int max_pages,
           int page_tokens, cudaStream_t st) {
    launch_k(embed_kernel, dim3(max_rows), dim3(128), 0, st, meta, emb, gain, x, xb, ss_a, d, last_token, page_table,
             max_pages, page_tokens);
}

// Prefill: token ids come staged per token.
__global__ void embed_tokens_kernel(const int32_t* __restrict__ tokens, const int* __restrict__ n_tokens,
                                    const __nv_bfloat16* __restrict__ emb, float* __restrict__ x, int d) {
    const int row = blockIdx.x;
    if (row >= *n_tokens) return;
    const int tok = tokens[row];
    const uint4* src = reinterpret_cast<const uint4*>(emb + static_cast<int64_t>(tok) * d);
    float4* dst = reinterpret_cast<float4*>(x + static_cast<int64_t>(row) * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
        const uint4 v = src[i];
        dst[2 * i] = make_float4(bf_lo(v.x), bf_hi(v.x), bf_lo(v.y), bf_hi(v.y));
        dst[2 * i + 1] = make_float4(bf_lo(v.z), bf_hi(v.z), bf_lo(v.w), bf_hi(v.w));
    }
}
void embed_tokens(const int32_t* tokens, const int* n_tokens_dev, int rows, const __nv_bfloat16* emb, float* x, int d,
                  cudaStream_t st) {
    embed_tokens_kernel<<<rows, 128, 0, st>>>(tokens, n_tokens_dev, emb, x, d);
    SW_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- RMSNorm
// One CTA per row, the row held in registers (VPT float4 per thread): one HBM
// read of x, fp32 statistics, bf16 output feeding the next GEMM.
// `rows_dev` (optional) bounds the live rows at run time (graph-safe);
// `row_index` (optional) gathers rows (LM head on the last prompt position).
template <int VPT>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                               __nv_bfloat16* __restrict__ y, int d, float eps, const int* rows_dev,
                               const int32_t* __restrict__ row_index) {
    const int row = blockIdx.x;
    if (rows_dev && row >= *rows_dev) return;
    const int src_row = row_index ? row_index[row] : row;
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<int64_t>(src_row) * d);
    float4 v[VPT];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        v[k] = i < d / 4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
    __shared__ float red[32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / static_cast<float>(d) + eps);
    const uint2* g2 = reinterpret_cast<const uint2*>(g);
    uint2* y2 = reinterpret_cast<uint2*>(y + static_cast<int64_t>(row) * d);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= d / 4) break;
        const uint2 gg = g2[i];
        uint2 o;
        o.x = pack_bf2(v[k].x * inv * bf_lo(gg.x), v[k].y * inv * bf_hi(gg.x));
        o.y = pack_bf2(v[k].z * inv * bf_lo(gg.y), v[k].w * inv * bf_hi(gg.y));
        y2[i] = o;
    }
}

void rmsnorm(const float* x, const __nv_bfloat16* g, __nv_bfloat16* y, int rows, int d, float eps, const int* rows_dev,
             const int32_t* row_index, cudaStream_t st) {
    const int threads = std::min(256, std::max(32, d / 4));
    const int vpt = cdiv(d / 4, threads);
    if (vpt <= 1) rmsnorm_kernel<1><<<rows, threads, 0, st>>>(x, g, y, d, eps, rows_dev, row_index);
    else if (vpt <= 2) rmsnorm_kernel<2><<<rows, threads, 0, st>>>(x, g, y, d, eps, rows_dev, row_index);
    else if (vpt <= 4) rmsnorm_kernel<4><<<rows, threads, 0, st>>>(x, g, y, d, eps, rows_dev, row_index);
    else if (vpt <= 8) rmsnorm_kernel<8><<<rows, threads, 0, st>>>(x, g, y, d, eps, rows_dev, row_index);
    else throw_cuda("rmsnorm: d_model too large", cudaErrorInvalidValue, __FILE__, __LINE__);
    SW_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- RoPE + KV
// qkv fp32 [T, (H + 2 Hkv) * hd] (GEMM output, kept fp32 so q/k are rounded to
// bf16 once, after the rotation) -> q [T, H*hd] roped, and K (roped)
// / V scattered into the paged cache of layer `layer`:
//   pages[layer][page][kv][head][page_tokens][hd],  page = table[slot][pos / B].
// cos/sin of pos * inv_freq[i] for every position < max_pos: the same fp32
// angle and sincosf as computing it inline, evaluated once per model.
__global__ void rope_table_kernel(const float* __restrict__ inv_freq, float2* __restrict__ table, int max_pos,
                                  int half) {
    const int64_t n = static_cast<int64_t>(max_pos) * half;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int pos = static_cast<int>(k / half), i = static_cast<int>(k % half);
        float s, c;
        sincosf(static_cast<float>(pos) * inv_freq[i], &s, &c);
        table[k] = make_float2(c, s);
    }
}
void rope_table(const float* inv_freq, float2* table, int max_pos, int half, cudaStream_t st) {
    rope_table_kernel<<<148 * 4, 256, 0, st>>>(inv_freq, table, max_pos, half);
    SW_LAUNCH_CHECK();
}

__global__ void rope_kv_kernel(const float* __restrict__ qkv, kv_t* __restrict__ q_out,
                               kv_t* __restrict__ kv_layer, const int32_t* __restrict__ tok_pos,
                               const int32_t* __restrict__ tok_slot, const int32_t* __restrict__ page_table,
                               const float2* __restrict__ cs_table, int rows, const int* rows_dev, int H, int Hkv,
                               int hd, int max_pages, int page_tokens, int64_t page_stride) {
    const int t = blockIdx.x;
    const int live = rows_dev ? *rows_dev : rows;
    if (t >= live) return;
    const int half = hd / 2;
    const int pos = tok_pos[t];
    const int slot = tok_slot[t];
    const int page = page_table[static_cast<int64_t>(slot) * max_pages + pos / page_tokens];
    const int off = pos % page_tokens;
    const int width = (H + 2 * Hkv) * hd;
    const float* src = qkv + static_cast<int64_t>(t) * width;
    kv_t* kbase = kv_layer + static_cast<int64_t>(page) * page_stride;
    const int64_t head_stride = static_cast<int64_t>(page_tokens) * hd;
    const int64_t kv_stride = static_cast<int64_t>(Hkv) * head_stride;
    // (head, i) pairs over q and k heads: rotate; v heads: copy.
    for (int idx = threadIdx.x; idx < (H + Hkv) * half; idx += blockDim.x) {
        const int h = idx / half, i = idx % half;
        const float2 cs = cs_table[static_cast<int64_t>(pos) * half + i];
        const float c = cs.x, s = cs.y;
        const float a = src[h * hd + i], b = src[h * hd + i + half];
        const kv_t ra = __float2half_rn(a * c - b * s);
        const kv_t rb = __float2half_rn(b * c + a * s);
        if (h < H) {
            kv_t* qd = q_out + static_cast<int64_t>(t) * H * hd + h * hd;
            qd[i] = ra;
            qd[i + half] = rb;
        } else {
            kv_t* kd = kbase + (h - H) * head_stride + off * hd;
            kd[i] = ra;
            kd[i + half] = rb;
        }
    }
    for (int idx = threadIdx.x; idx < Hkv * hd; idx += blockDim.x) {
        const int h = idx / hd, i = idx % hd;
        kbase[kv_stride + h * head_stride + off * hd + i] = __float2half_rn(src[(H + Hkv + h) * hd + i]);
    }
}

void rope_kv(const float* qkv, kv_t* q_out, kv_t* kv_layer, const int32_t* tok_pos,
             const int32_t* tok_slot, const int32_t* page_table, const float2* cs_table, int rows, const int* rows_dev,
             int H, int Hkv, int hd, int max_pages, int page_tokens, cudaStream_t st) {
    const int64_t page_stride = 2LL * Hkv * page_tokens * hd;
    rope_kv_kernel<<<rows, 256, 0, st>>>(qkv, q_out, kv_layer, tok_pos, tok_slot, page_table, cs_table, rows,
                                         rows_dev, H, Hkv, hd, max_pages, page_tokens, page_stride);
    SW_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- tokens
// Decode the packed argmax keys of `rows` rows into the slots' last token and
// output buffer, then reset the keys for the next launch.
__global__ void finalize_tokens_kernel(unsigned long long* __restrict__ keys, const int32_t* __restrict__ slot,
                                       const int32_t* __restrict__ out_index, int rows, const int* rows_dev,
                                       int32_t* __restrict__ last_token, int32_t* __restrict__ out_tokens,
                                       int max_out) {
    griddep_launch_dependents();
    griddep_wait();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int live = rows_dev ? *rows_dev : rows;
    if (r >= rows) return;
    if (r < live) {
        const int tok = static_cast<int>(argmax_index(keys[r]));
        const int s = slot[r];
        last_token[s] = tok;
        const int oi = out_index[r];
        if (oi >= 0 && oi < max_out) out_tokens[static_cast<int64_t>(s) * max_out + oi] = tok;
    }
    keys[r] = 0ull;
}

void finalize_tokens(unsigned long long* keys, const int32_t* slot, const int32_t* out_index, int rows,
                     const int* rows_dev, int32_t* last_token, int32_t* out_tokens, int max_out, cudaStream_t st) {
    launch_k(finalize_tokens_kernel, dim3(cdiv(rows, 128)), dim3(128), 0, st, keys, slot, out_index, rows, rows_dev,
             last_token, out_tokens, max_out);
}

}  // namespace sw

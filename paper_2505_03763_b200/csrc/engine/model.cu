// Model runtime: weights, KV arena, the prefill and decode forward passes, and
// the kernel-level C-ABI (sw_model_create ... sw_decode_enqueue).
//
// These two passes are what replaces the reference's task pricing
// (make_prompt_task / make_token_step_task, splitsim/gpu_model.hpp:154-189):
// a prompt task runs prefill_forward over the batch's prompts, a token step
// runs decode_forward over the running batch.
//
// HBM layout (bf16 unless noted):
//   weights  one arena; per layer wqkv [(H+2Hkv)hd, d], wo [d, H hd],
//            wgu [2 ffn, d] in [gate 64 | up 64] row blocks (SwiGLU fuses into
//            the GEMM epilogue), wd [d, ffn]; embedding [V, d]; LM head [V, d]
//            (aliases the embedding when tied).
//   KV       pages[L][n_pages][K|V][Hkv][16 tokens][hd] fp16: a (layer, page, head)
//            is one contiguous 16 x hd block, so attention reads whole pages
//            with 16 B vector loads; page ids come from per-slot page tables
//            (int32 [slots][max_pages]) shared by both phases -- the prompt
//            writes the pages, the decode steps read them, nothing is copied
//            at the phase handoff.
// Decode steps are captured into one CUDA graph per row bucket; the graph
// reads the live row count and per-row metadata from a device StepMeta the
// host refreshes with a single H2D copy per step.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../host/capi_util.hpp"
#include "../kernels/attention.cuh"
#include "../kernels/common.cuh"
#include "../kernels/elementwise.cuh"
#include "../kernels/gemm_sm100.cuh"
#include "model.hpp"
#include "partition.hpp"

namespace sw {

extern std::atomic<unsigned long long> g_launches;

namespace {

constexpr int kLmRowsMax = 256;  // LM-head rows per GEMM pass (swap-AB N <= 256)
constexpr int kLmBufRows = 512;  // LM-head rows per forward (a fused mixed step: prompts + up to 256 decode rows)
constexpr int kSplitTiles = 640;     // split-K scratch: (tiles x splits) capacity
constexpr int kSplitCounters = 1024;
constexpr int kSsParts = 64;  // sum(x^2) partial rows per norm (d_model / 128 <= 64)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <class T>
T* dalloc(size_t n) {
    void* p = nullptr;
    SW_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

void ring_init(PinnedRing& r, int n, size_t bytes) {
    r.bytes = bytes;
    for (int i = 0; i < n; ++i) {
        void* p = nullptr;
        SW_CUDA(cudaMallocHost(&p, bytes));
        cudaEvent_t e;
        SW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        SW_CUDA(cudaEventRecord(e, 0));
        r.slots.push_back(p);
        r.done.push_back(e);
    }
}

// Claim the next staging slot (waits only if its previous copy is still pending).
void* ring_claim(PinnedRing& r, int& idx) {
    idx = r.next;
    r.next = (r.next + 1) % static_cast<int>(r.slots.size());
    SW_CUDA(cudaEventSynchronize(r.done[idx]));
    return r.slots[idx];
}

void ring_release(PinnedRing& r, int idx, cudaStream_t st) { SW_CUDA(cudaEventRecord(r.done[idx], st)); }

void ws_alloc(Workspace& w, const sw_model_desc& d, int rows, bool decode, int max_splits_cap) {
    const int qkv_w = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
    w.rows = rows;
    w.x = dalloc<float>(static_cast<size_t>(rows) * d.d_model);
    w.xn = dalloc<__nv_bfloat16>(static_cast<size_t>(rows) * d.d_model);
    w.qkv = dalloc<float>(static_cast<size_t>(rows) * qkv_w);
    w.q = dalloc<kv_t>(static_cast<size_t>(rows) * d.n_heads * d.head_dim);
    w.attn = dalloc<__nv_bfloat16>(static_cast<size_t>(rows) * d.n_heads * d.head_dim);
    w.act = dalloc<__nv_bfloat16>(static_cast<size_t>(rows) * d.ffn_dim);
    w.xlast = dalloc<__nv_bfloat16>(static_cast<size_t>(kLmBufRows) * d.d_model);
    w.keys = dalloc<unsigned long long>(kLmBufRows);
    SW_CUDA(cudaMemset(w.keys, 0, kLmBufRows * sizeof(unsigned long long)));
    SW_CUDA(cudaMemset(w.x, 0, static_cast<size_t>(rows) * d.d_model * sizeof(float)));
    SW_CUDA(cudaMemset(w.xn, 0, static_cast<size_t>(rows) * d.d_model * 2));
    SW_CUDA(cudaMemset(w.attn, 0, static_cast<size_t>(rows) * d.n_heads * d.head_dim * 2));
    SW_CUDA(cudaMemset(w.act, 0, static_cast<size_t>(rows) * d.ffn_dim * 2));
    if (decode) {
        w.meta = dalloc<StepMeta>(1);
        SW_CUDA(cudaMemset(w.meta, 0, sizeof(StepMeta)));
        w.ss = dalloc<float>(2 * kSsParts * kSsStride);
        SW_CUDA(cudaMemset(w.ss, 0, 2 * kSsParts * kSsStride * sizeof(float)));
        const int G = d.n_heads / d.n_kv_heads;
        const size_t parts = static_cast<size_t>(kMaxDecodeRows) * d.n_kv_heads * max_splits_cap * G;
        w.part_o = dalloc<float>(parts * d.head_dim);
        w.part_ml = dalloc<float>(parts * 2);
        int dev = 0, sms = 0;
        SW_CUDA(cudaGetDevice(&dev));
        SW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const size_t flat = attn_decode_flat_part_rows(sms) * G;
        w.flat_o = dalloc<float>(flat * d.head_dim);
        w.flat_ml = dalloc<float>(flat * 2);
        w.attn_cnt = dalloc<unsigned>(static_cast<size_t>(kMaxDecodeRows) * d.n_kv_heads);
        SW_CUDA(cudaMemset(w.attn_cnt, 0, static_cast<size_t>(kMaxDecodeRows) * d.n_kv_heads * sizeof(unsigned)));
        w.splitk_floats = static_cast<size_t>(kSplitTiles) * 256 * 128;
        w.splitk_ws = dalloc<float>(w.splitk_floats);
        w.splitk_cnt = dalloc<unsigned>(kSplitCounters);
        SW_CUDA(cudaMemset(w.splitk_cnt, 0, kSplitCounters * sizeof(unsigned)));
    } else {
        // header + tokens/pos/slot per token + per-seq arrays + tiles + page rows
        const size_t T = static_cast<size_t>(rows);
        w.pmeta_bytes =
            (16 + 3 * T + 6 * (T + 1) + 2 * (T / 64 + T + 1) + 2 * (T / 128 + T + 1) + (T / 16 + T + 1)) * sizeof(int32_t);
        w.pmeta = dalloc<int32_t>(w.pmeta_bytes / sizeof(int32_t));
    }
}

GemmProblem gp(const void* X, int64_t x_rows, const void* W, int64_t w_rows, int tokens, int features, int K,
               int mode, bool swap, void* out, int ldo, const int* live = nullptr, const Workspace* ws = nullptr) {
    GemmProblem p{};
    if (ws && ws->splitk_ws) {
        p.ws = ws->splitk_ws;
        p.ws_floats = ws->splitk_floats;
        p.counters = ws->splitk_cnt;
        p.n_counters = kSplitCounters;
    }
    p.X = X;
    p.x_rows = x_rows;
    p.W = W;
    p.w_rows = w_rows;
    p.tokens = tokens;
    p.live_tokens = live;
    p.features = features;
    p.K = K;
    p.mode = mode;
    p.swap = swap;
    p.out = out;
    p.ldo = ldo;
    return p;
}

// install staged page-table rows: rows packed back to back, offsets per seq
__global__ void install_pages_kernel(const int32_t* __restrict__ rows, const int32_t* __restrict__ off,
                                     const int32_t* __restrict__ seq_slot, int32_t* __restrict__ table,
                                     int max_pages) {
    const int s = blockIdx.x;
    const int b = off[s], e = off[s + 1];
    int32_t* dst = table + static_cast<int64_t>(seq_slot[s]) * max_pages;
    for (int i = threadIdx.x; i < e - b; i += blockDim.x) dst[i] = rows[b + i];
}

void lm_head(sw_model* m, Workspace& w, int rows, const int* live, float* logits_out, cudaStream_t st) {
    const sw_model_desc& d = m->desc;
    // passes of <= 256 rows (the swap-AB N bound); `live` (graph-captured decode) implies rows <= 256
    for (int r0 = 0; r0 < rows; r0 += kLmRowsMax) {
        const int n = std::min(kLmRowsMax, rows - r0);
        const __nv_bfloat16* x = w.xlast + static_cast<size_t>(r0) * d.d_model;
        GemmProblem p = gp(x, kLmRowsMax, m->lm, d.vocab, n, d.vocab, d.d_model, EPI_ARGMAX, true, nullptr, 0, live);
        p.argmax = w.keys + r0;
        gemm_run(p, st);
        if (logits_out) {
            GemmProblem q = gp(x, kLmRowsMax, m->lm, d.vocab, n, d.vocab, d.d_model, EPI_STORE_F32, true,
                               logits_out + static_cast<int64_t>(r0) * d.vocab, d.vocab, live);
            gemm_run(q, st);
        }
    }
}

}  // namespace

int decode_bucket(int n) {
    static const int kBuckets[] = {1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 160, 192, 224, 256};
    for (int b : kBuckets)
        if (n <= b) return b;
    throw ContractViolation("decode: batch of " + std::to_string(n) + " rows exceeds 256");
}

// ------------------------------------------------------------------ prefill
namespace {
void prefill_chunk(sw_model* m, sw_kv* kv, const sw_batch& b, int first, int last, int64_t tok_off, int64_t page_off,
                   const sw_batch* dec, float* logits_out, cudaStream_t st, bool lean, int yield_tiles);
}  // namespace

void prefill_forward(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st, bool lean, int yield_tiles) {
    const sw_model_desc& d = m->desc;
    Workspace& w = m->pre;
    const int B = kv->page_tokens;
    // Split the batch into chunks of whole prompts that fit the workspace.
    int first = 0;
    int64_t tok_off = 0, page_off = 0;
    while (first < b.n) {
        int last = first, T = 0;
        while (last < b.n && T + b.n_tokens[last] <= w.rows && last - first < kLmRowsMax) T += b.n_tokens[last++];
        if (last == first)
            throw ConfigError("prefill: prompt of " + std::to_string(b.n_tokens[first]) +
                              " tokens exceeds model.max_prefill_tokens=" + std::to_string(w.rows));
        prefill_chunk(m, kv, b, first, last, tok_off, page_off, nullptr,
                      b.logits_out ? b.logits_out + static_cast<int64_t>(first) * d.vocab : nullptr, st, lean,
                      yield_tiles);
        for (int r = first; r < last; ++r) {
            tok_off += b.n_tokens[r];
            page_off += cdiv((b.positions ? b.positions[r] : 0) + b.n_tokens[r], B);
        }
        first = last;
    }
}

// ------------------------------------------------------------------ decode
namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

DecodeAttnArgs decode_attn_args(const sw_model* m, const sw_kv* kv, const Workspace& w) {
    const sw_model_desc& d = m->desc;
    DecodeAttnArgs aa{};
    aa.meta = w.meta;
    aa.page_table = kv->page_table;
    aa.max_pages = kv->max_pages;
    aa.page_tokens = kv->page_tokens;
    aa.page_stride = kv->page_stride;
    aa.kv_stride = kv->page_stride / 2;
    aa.H = d.n_heads;
    aa.Hkv = d.n_kv_heads;
    aa.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d.head_dim)));
    aa.chunk = kv->chunk;
    aa.max_splits = kv->max_splits;
    aa.part_o = w.part_o;
    aa.part_ml = w.part_ml;
    aa.counters = w.attn_cnt;
    static const int target = env_int("SW_ATTN_CTAS", 296);
    aa.target_ctas = target;
    aa.max_ctx = kv->max_pages * kv->page_tokens;
    return aa;
}

DecodeFlatArgs decode_flat_args(const sw_model* m, const sw_kv* kv, const Workspace& w) {
    const sw_model_desc& d = m->desc;
    DecodeFlatArgs fa{};
    fa.meta = w.meta;
    fa.page_table = kv->page_table;
    fa.max_pages = kv->max_pages;
    fa.H = d.n_heads;
    fa.Hkv = d.n_kv_heads;
    fa.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d.head_dim)));
    fa.page_rows = static_cast<int>(kv->page_stride / d.head_dim);
    fa.v_rows = static_cast<int>(kv->page_stride / 2 / d.head_dim);
    fa.part_o = w.flat_o;
    fa.part_ml = w.flat_ml;
    fa.counters = w.attn_cnt;
    return fa;
}

void decode_layers(sw_model* m, sw_kv* kv, int R, cudaStream_t st, int lane, bool use_flat) {
    // One decode step, 5 kernels per layer, chained with programmatic dependent
    // launch (each kernel's weight stream starts while its predecessor drains):
    //   qkv  GEMM . RMSNorm scale . RoPE -> q, K/V straight into the paged cache
    //   attn split-KV paged attention
    //   wo   GEMM + residual; emits bf16(x) and sum(x^2) for the next norm
    //   gu   GEMM . RMSNorm scale . SwiGLU
    //   wd   GEMM + residual; emits bf16(x) and sum(x^2)
    // RMSNorm is folded into the consuming GEMM: its B operand is bf16(x * g)
    // (written by the producer with the consuming norm's gain g) and the
    // epilogue scales by rsqrt(mean(x^2) + eps).
    PdlScope pdl(true);
    const sw_model_desc& d = m->desc;
    Workspace& w = m->dec[lane];
    const int* live = &w.meta->n;
    const int qkv_w = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
    const int hdH = d.n_heads * d.head_dim;
    float* ss_a = w.ss;  // [kSsParts][kSsStride] partial sum(x^2) rows
    float* ss_b = w.ss + kSsParts * kSsStride;
    const int parts = d.d_model / 128;  // one partial row per feature tile of a residual GEMM
    __nv_bfloat16* xb = w.xn;
    embed(w.meta, R, m->emb, m->layers[0].g_attn, w.x, xb, ss_a, d.d_model, kv->last_token, kv->page_table,
          kv->max_pages, kv->page_tokens, st);
    DecodeAttnArgs aa = decode_attn_args(m, kv, w);
    auto norm_in = [&](GemmProblem& p, const float* ss, int nparts) {
        p.fx.ss_parts = ss;
        p.fx.ss_nparts = nparts;
        p.fx.norm_dim = d.d_model;
        p.fx.norm_eps = d.norm_eps;
    };
    auto resid_out = [&](GemmProblem& p, float* ss_out, const __nv_bfloat16* next_gain) {
        p.fx.x_bf16 = xb;
        p.fx.x_gain = next_gain;
        p.fx.ss_part_out = ss_out;
    };
    static const int ablate = env_int("SW_ABLATE", 0);  // timing experiments only: skip kernel classes
    DecodeFlatArgs fa{};
    const int flat_ctas = stream_sm_count(st);
    if (use_flat) fa = decode_flat_args(m, kv, w);
    for (int l = 0; l < d.n_layers; ++l) {
        const LayerWeights& L = m->layers[l];
        kv_t* kvl = kv->pages + l * kv->layer_stride;
        GemmProblem pq = gp(xb, w.rows, L.wqkv, qkv_w, R, qkv_w, d.d_model, EPI_QKV_ROPE, true, nullptr, qkv_w, live, &w);
        norm_in(pq, ss_a, l == 0 ? 1 : parts);
        pq.fx.pos = w.meta->pos;
        pq.fx.slot = w.meta->slot;
        pq.fx.page_table = kv->page_table;
        pq.fx.max_pages = kv->max_pages;
        pq.fx.page_tokens = kv->page_tokens;
        pq.fx.rope_cs = m->rope_cs;
        pq.fx.q_out = w.q;
        pq.fx.kv_layer = kvl;
        pq.fx.page_stride = kv->page_stride;
        pq.fx.H = d.n_heads;
        pq.fx.Hkv = d.n_kv_heads;
        pq.fx.hd = d.head_dim;
        if (!(ablate & 2)) gemm_run(pq, st);
        if (!(ablate & 1)) {
            if (use_flat) {
                fa.layer_row0 = static_cast<int>(l * kv->layer_stride / d.head_dim);
                attn_decode_flat(kv->tm_kv, w.q, w.attn, fa, flat_ctas, d.head_dim, d.n_heads / d.n_kv_heads, st);
            } else {
                attn_decode(w.q, kvl, w.attn, aa, R, d.head_dim, st);
            }
        }
        GemmProblem po = gp(w.attn, w.rows, L.wo, d.d_model, R, d.d_model, hdH, EPI_RESID, true, w.x, d.d_model, live, &w);
        resid_out(po, ss_b, L.g_mlp);
        if (!(ablate & 4)) gemm_run(po, st);
        GemmProblem pg = gp(xb, w.rows, L.wgu, 2 * d.ffn_dim, R, 2 * d.ffn_dim, d.d_model, EPI_SWIGLU, true, w.act,
                            d.ffn_dim, live, &w);
        norm_in(pg, ss_b, parts);
        if (!(ablate & 8)) gemm_run(pg, st);
        GemmProblem pd = gp(w.act, w.rows, L.wd, d.d_model, R, d.d_model, d.ffn_dim, EPI_RESID, true, w.x, d.d_model,
                            live, &w);
        resid_out(pd, ss_a, l + 1 < d.n_layers ? m->layers[l + 1].g_attn : m->g_final);
        if (!(ablate & 16)) gemm_run(pd, st);
    }
    GemmProblem pl = gp(xb, w.rows, m->lm, d.vocab, R, d.vocab, d.d_model, EPI_ARGMAX, true, nullptr, 0, live);
    pl.argmax = w.keys;
    norm_in(pl, ss_a, parts);  // argmax is scale invariant; kept so logits and argmax see one definition
    if (!(ablate & 32)) gemm_run(pl, st);
    finalize_tokens(w.keys, w.meta->slot, w.meta->out_index, R, live, kv->last_token, kv->out_tokens, kv->max_out, st);
}


}  // namespace

// Stage one decode step's metadata (StepMeta, one H2D copy) on `lane` and pick its attention kernel;
// returns the row bucket.
static int stage_decode(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st, int lane, bool& flat) {
    const sw_model_desc& d = m->desc;
    if (lane < 0 || lane >= sw_model::kMaxDecodeLanes) throw ContractViolation("decode: lane out of range");
    Workspace& w = m->dec[lane];
    if (!w.x) ws_alloc(w, d, std::min(d.max_decode_batch, kMaxDecodeRows), true, 16);  // lanes > 0 on first use
    if (m->dec_ring[lane].slots.empty()) ring_init(m->dec_ring[lane], 8, sizeof(StepMeta));
    if (b.n < 1 || b.n > kMaxDecodeRows) throw ContractViolation("decode: batch size out of range");
    if (b.n > w.rows) throw ConfigError("decode: batch exceeds model.max_decode_batch");
    int idx;
    StepMeta* h = static_cast<StepMeta*>(ring_claim(m->dec_ring[lane], idx));
    h->n = b.n;
    for (int i = 0; i < b.n; ++i) {
        const int slot = b.slots[i], pos = b.positions[i];
        if (slot < 0 || slot >= kv->n_slots) throw ContractViolation("decode: slot out of range");
        if (pos < 0 || pos >= kv->max_pages * kv->page_tokens) throw ContractViolation("decode: position out of range");
        h->slot[i] = slot;
        h->pos[i] = pos;
        h->token[i] = b.tokens ? b.tokens[i] : -1;
        h->new_page[i] = b.new_page ? b.new_page[i] : -1;
        if (h->new_page[i] >= kv->n_pages) throw ContractViolation("decode: page id out of range");
        h->out_index[i] = b.out_index ? b.out_index[i] : -1;
    }
    const size_t bytes = offsetof(StepMeta, slot) + sizeof(StepMeta::slot) * 5;
    SW_CUDA(cudaMemcpyAsync(w.meta, h, bytes, cudaMemcpyHostToDevice, st));
    count_transfer(bytes, 0);
    ring_release(m->dec_ring[lane], idx, st);
    const int R = std::min(decode_bucket(b.n), w.rows);
    // decode attention kernel: the flat page-balanced one for long contexts, the per-unit
    // split-KV one below (its independent CTAs flow around concurrent prefill work);
    // SW_ATTN_FLAT=0/1 forces one (profiles/r01c/attn_flat_sweep.txt)
    static const int flat_env = env_int("SW_ATTN_FLAT", 2);
    static const int flat_ctx = env_int("SW_ATTN_FLAT_CTX", 2048);
    flat = false;
    if (kv->tm_kv_ok && flat_env == 1) {
        flat = true;
    } else if (kv->tm_kv_ok && flat_env == 2) {
        // long contexts, or too few (row, kv head) units for the per-unit kernel to fill two CTAs per SM
        // without splitting them (Llama-1B b=32 ctx 576: 0.970 -> 0.881 ms per step)
        long long ctx = 0;
        for (int i = 0; i < b.n; ++i) ctx += b.positions[i] + 1;
        flat = ctx >= static_cast<long long>(flat_ctx) * b.n || b.n * d.n_kv_heads <= 2 * stream_sm_count(st);
    }
    return R;
}

void decode_forward(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st, bool use_graph, int lane, int lanes) {
    const sw_model_desc& d = m->desc;
    bool flat = false;
    const int R = stage_decode(m, kv, b, st, lane, flat);
    Workspace& w = m->dec[lane];
    auto run = [&](cudaStream_t s) {
        decode_layers(m, kv, R, s, lane, flat);
    };
    DecodeGraph& g = m->graphs[{kv, R, lane | (flat ? 32 : 0), stream_partition_tag(st)}];
    if (use_graph && g.exec) {
        SW_CUDA(cudaGraphLaunch(g.exec, st));
        count_launches(g.kernels);
    } else {
        run(st);
        if (use_graph && ++g.eager_runs >= 1) {
            // capture once the kernels' attributes are configured (first eager run), on the
            // launch stream itself: the graph then runs in that stream's (green) context
            // (the legacy default stream cannot capture: use a scratch stream of the primary context)
            const bool legacy = st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread;
            cudaStream_t cs = st;
            if (legacy) SW_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t graph;
            SW_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            const unsigned long long before = g_launches.load();
            run(cs);
            g.kernels = g_launches.load() - before;
            g_launches.fetch_sub(g.kernels);  // captured, not launched
            SW_CUDA(cudaStreamEndCapture(cs, &graph));
            SW_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
            SW_CUDA(cudaGraphDestroy(graph));
            if (legacy) SW_CUDA(cudaStreamDestroy(cs));
        }
    }
    if (b.logits_out) {  // parity checks: fp32 logits from the same folded-norm input
        GemmProblem q = gp(w.xn, w.rows, m->lm, d.vocab, b.n, d.vocab, d.d_model, EPI_STORE_F32, true,
                           b.logits_out, d.vocab);
        q.fx.ss_parts = w.ss;
        q.fx.ss_nparts = d.d_model / 128;
        q.fx.norm_dim = d.d_model;
        q.fx.norm_eps = d.norm_eps;
        gemm_run(q, st);
    }
}

// One decode step's attention alone -- every layer's launch of the kernel the step would pick -- over
// the rows' paged contexts (bench.py: the roofline of the dominant kernel of a decode-heavy run; the
// q rows are whatever the workspace holds, the KV reads are the step's).
static void decode_attention_only(sw_model* m, sw_kv* kv, const sw_batch& b, cudaStream_t st) {
    bool flat = false;
    const int R = stage_decode(m, kv, b, st, 0, flat);
    const sw_model_desc& d = m->desc;
    PdlScope pdl(true);
    Workspace& w = m->dec[0];
    DecodeAttnArgs aa = decode_attn_args(m, kv, w);
    DecodeFlatArgs fa = decode_flat_args(m, kv, w);
    const int flat_ctas = stream_sm_count(st);
    for (int l = 0; l < d.n_layers; ++l) {
        kv_t* kvl = kv->pages + l * kv->layer_stride;
        if (flat) {
            fa.layer_row0 = static_cast<int>(l * kv->layer_stride / d.head_dim);
            attn_decode_flat(kv->tm_kv, w.q, w.attn, fa, flat_ctas, d.head_dim, d.n_heads / d.n_kv_heads, st);
        } else {
            attn_decode(w.q, kvl, w.attn, aa, R, d.head_dim, st);
        }
    }
}

// ------------------------------------------------------------------ prefill chunk / fused mixed step
namespace {

// One launch over prompts [first, last) of b (all fit the workspace), plus --
// for a fused mixed step -- the decode rows of `dec` appended after the prompt
// tokens: every projection GEMM runs once over [prompt tokens | decode rows].
void prefill_chunk(sw_model* m, sw_kv* kv, const sw_batch& b, int first, int last, int64_t tok_off, int64_t page_off,
                   const sw_batch* dec, float* logits_out, cudaStream_t st, bool lean, int yield_tiles) {
    const sw_model_desc& d = m->desc;
    auto lp = [lean, yield_tiles](GemmProblem p) {
        p.lean = lean;
        p.yield_tiles = yield_tiles;
        return p;
    };
    Workspace& w = m->pre;
    const int B = kv->page_tokens;
    const int D = dec ? dec->n : 0;  // fused decode rows
    int Tp = 0;
    for (int r = first; r < last; ++r) Tp += b.n_tokens[r];
    const int T = Tp + D;
    const int S = last - first;
    const int NL = S + D;  // LM-head rows: every prompt's last position, then the decode rows
    // ---- stage metadata (one H2D copy)
    int idx;
    int32_t* h = static_cast<int32_t*>(ring_claim(m->pre_ring, idx));
    int32_t* p = h + 16;
    auto take = [&](int n) {
        int32_t* q = p;
        p += n;
        return q;
    };
    int32_t *tokens = take(Tp), *tpos = take(T), *tslot = take(T), *cu = take(S + 1), *sslot = take(NL),
            *lastrow = take(NL), *oidx = take(NL), *poff = take(S + 1), *spos0 = take(S);
    // chunked prefill: prompt r covers positions [pos0, pos0 + n) of its sequence; its earlier positions are
    // already in the paged KV cache (keys [0, pos0 + q] for query position pos0 + q)
    const int32_t* pos0_of = b.positions;
    int n_tiles = 0;
    for (int s = 0; s < S; ++s) n_tiles += cdiv(b.n_tokens[first + s], 64);
    int32_t *tseq = take(n_tiles), *tq0 = take(n_tiles);
    int n_tiles128 = 0;  // 128-row tiles of the tcgen05 attention
    for (int s = 0; s < S; ++s) n_tiles128 += cdiv(b.n_tokens[first + s], 128);
    int32_t *tseq128 = take(n_tiles128), *tq0128 = take(n_tiles128);
    int n_pages_total = 0;
    for (int s = 0; s < S; ++s) n_pages_total += cdiv((pos0_of ? pos0_of[first + s] : 0) + b.n_tokens[first + s], B);
    int32_t* prow = take(n_pages_total);
    int t = 0, ti = 0, ti128 = 0, pg = 0;
    cu[0] = 0;
    poff[0] = 0;
    for (int s = 0; s < S; ++s) {
        const int r = first + s, n = b.n_tokens[r];
        const int p0 = pos0_of ? pos0_of[r] : 0;
        if (b.slots[r] < 0 || b.slots[r] >= kv->n_slots) throw ContractViolation("prefill: slot out of range");
        if (n < 1) throw ContractViolation("prefill: empty prompt");
        if (p0 < 0 || p0 % 128 != 0) throw ContractViolation("prefill: a prompt chunk must start at a multiple of 128");
        const int np = cdiv(p0 + n, B);
        if (np > kv->max_pages) throw ContractViolation("prefill: prompt exceeds the slot's page-table row");
        for (int j = 0; j < n; ++j) {
            tokens[t + j] = b.tokens[tok_off + j];
            if (tokens[t + j] < 0 || tokens[t + j] >= d.vocab) throw ContractViolation("prefill: token out of range");
            tpos[t + j] = p0 + j;
            tslot[t + j] = b.slots[r];
        }
        for (int j = 0; j < np; ++j) {
            const int pid = b.page_rows[page_off + j];
            if (pid < 0 || pid >= kv->n_pages) throw ContractViolation("prefill: page id out of range");
            prow[pg + j] = pid;
        }
        for (int q0 = 0; q0 < n; q0 += 64, ++ti) {
            tseq[ti] = s;
            tq0[ti] = q0;
        }
        for (int q0 = 0; q0 < n; q0 += 128, ++ti128) {
            tseq128[ti128] = s;
            tq0128[ti128] = q0;
        }
        tok_off += n;
        page_off += np;
        t += n;
        pg += np;
        cu[s + 1] = t;
        poff[s + 1] = pg;
        spos0[s] = p0;
        sslot[s] = b.slots[r];
        lastrow[s] = t - 1;
        oidx[s] = b.out_index ? b.out_index[r] : 0;
    }
    // fused decode rows: token rows [Tp, T) of every projection, their own positions and slots
    StepMeta* dm = nullptr;
    int dm_idx = -1;
    if (D > 0) {
        dm = static_cast<StepMeta*>(ring_claim(m->mix_ring, dm_idx));
        dm->n = D;
        for (int i = 0; i < D; ++i) {
            const int slot = dec->slots[i], pos = dec->positions[i];
            if (slot < 0 || slot >= kv->n_slots) throw ContractViolation("mixed step: slot out of range");
            if (pos < 0 || pos >= kv->max_pages * kv->page_tokens)
                throw ContractViolation("mixed step: position out of range");
            dm->slot[i] = slot;
            dm->pos[i] = pos;
            dm->token[i] = dec->tokens ? dec->tokens[i] : -1;
            dm->new_page[i] = dec->new_page ? dec->new_page[i] : -1;
            if (dm->new_page[i] >= kv->n_pages) throw ContractViolation("mixed step: page id out of range");
            dm->out_index[i] = dec->out_index ? dec->out_index[i] : -1;
            tpos[Tp + i] = pos;
            tslot[Tp + i] = slot;
            sslot[S + i] = slot;
            lastrow[S + i] = Tp + i;
            oidx[S + i] = dm->out_index[i];
        }
    }
    h[0] = Tp;
    h[1] = S;
    h[2] = n_tiles;
    h[3] = n_tiles128;
    const size_t bytes = static_cast<size_t>(p - h) * sizeof(int32_t);
    if (bytes > w.pmeta_bytes || bytes > m->pre_ring.bytes) throw ContractViolation("prefill: metadata overflow");
    SW_CUDA(cudaMemcpyAsync(w.pmeta, h, bytes, cudaMemcpyHostToDevice, st));
    count_transfer(bytes, 0);
    ring_release(m->pre_ring, idx, st);
    auto dev = [&](int32_t* hp) { return w.pmeta + (hp - h); };
    Workspace& mw = m->mix;
    if (D > 0) {
        const size_t mbytes = offsetof(StepMeta, slot) + sizeof(StepMeta::slot) * 5;
        SW_CUDA(cudaMemcpyAsync(mw.meta, dm, mbytes, cudaMemcpyHostToDevice, st));
        count_transfer(mbytes, 0);
        ring_release(m->mix_ring, dm_idx, st);
    }

    if (S > 0) {
        install_pages_kernel<<<S, 64, 0, st>>>(dev(prow), dev(poff), dev(sslot), kv->page_table, kv->max_pages);
        SW_LAUNCH_CHECK();
    }
    // ---- layers
    const int qkv_w = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
    const int hdH = d.n_heads * d.head_dim;
    if (Tp > 0) embed_tokens(dev(tokens), w.pmeta, Tp, m->emb, w.x, d.d_model, st);
    if (D > 0)  // decode rows: the slot's last token (device resident), new pages installed first
        embed(mw.meta, D, m->emb, m->layers[0].g_attn, w.x + static_cast<size_t>(Tp) * d.d_model,
              w.xn + static_cast<size_t>(Tp) * d.d_model, mw.ss, d.d_model, kv->last_token, kv->page_table,
              kv->max_pages, kv->page_tokens, st);
    PrefillAttnArgs aa{};
    aa.n_tiles = w.pmeta + 2;
    aa.tile_seq = dev(tseq);
    aa.tile_q0 = dev(tq0);
    aa.cu_seqlens = dev(cu);
    aa.seq_slot = dev(sslot);
    aa.page_table = kv->page_table;
    aa.max_pages = kv->max_pages;
    aa.page_tokens = B;
    aa.page_stride = kv->page_stride;
    aa.kv_stride = kv->page_stride / 2;
    aa.H = d.n_heads;
    aa.Hkv = d.n_kv_heads;
    aa.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d.head_dim)));
    // prefill attention on tcgen05 (SW_PREFILL_TC=0: the mma.sync kernel)
    static const int tc_env = env_int("SW_PREFILL_TC", 1);
    const bool use_tc = tc_env && kv->tm_kv_ok && (d.n_heads / d.n_kv_heads) % 2 == 0;  // head pairs share a kv head
    bool chunked = false;
    for (int s = 0; s < S && pos0_of; ++s) chunked |= pos0_of[first + s] > 0;
    if (chunked && !use_tc) throw ConfigError("prefill: prompt chunks past position 0 need the tcgen05 attention");
    // RoPE + KV write fused into the QKV GEMM epilogue (SW_PREFILL_ROPE_FUSED=0: separate rope_kv pass)
    static const int fuse_env = env_int("SW_PREFILL_ROPE_FUSED", 1);
    const bool fuse_rope = fuse_env != 0;
    PrefillTcArgs ta{};
    CUtensorMap tm_q{};
    // persistent prefill attention for short prompts (1B 32 x 512 layer: 165 -> 153 us); prompts of
    // many 128-row tiles keep one item per CTA (8B 4 x 8192: 4.37 vs 4.63 ms persistent)
    int max_prompt = 0;
    for (int s = 0; s < S; ++s) max_prompt = std::max(max_prompt, b.n_tokens[first + s]);
    const bool tc_persist = max_prompt <= 1024;
    if (use_tc) {
        ta.n_tiles = w.pmeta + 3;
        ta.tile_seq = dev(tseq128);
        ta.tile_q0 = dev(tq0128);
        ta.cu_seqlens = dev(cu);
        ta.seq_pos0 = dev(spos0);
        ta.seq_slot = dev(sslot);
        ta.page_table = kv->page_table;
        ta.max_pages = kv->max_pages;
        ta.H = d.n_heads;
        ta.Hkv = d.n_kv_heads;
        ta.scale_log2 = aa.scale_log2;
        ta.page_rows = static_cast<int>(kv->page_stride / d.head_dim);
        ta.v_rows = static_cast<int>(kv->page_stride / 2 / d.head_dim);
        tm_q = make_tmap_heads(w.q, static_cast<uint64_t>(w.rows), d.n_heads, d.head_dim);
    }
    // decode rows' attention: the decode kernels over their paged contexts (q and output rows from Tp on)
    DecodeAttnArgs da{};
    DecodeFlatArgs fa{};
    bool flat = false;
    const int R = D > 0 ? decode_bucket(D) : 0;
    if (D > 0) {
        da = decode_attn_args(m, kv, mw);
        long long ctx = 0;
        for (int i = 0; i < D; ++i) ctx += dec->positions[i] + 1;
        flat = kv->tm_kv_ok && (ctx >= 2048LL * D || D * d.n_kv_heads <= 2 * stream_sm_count(st));
        if (flat) fa = decode_flat_args(m, kv, mw);
    }
    kv_t* const q_dec = w.q + static_cast<size_t>(Tp) * hdH;
    __nv_bfloat16* const attn_dec = w.attn + static_cast<size_t>(Tp) * hdH;
    for (int l = 0; l < d.n_layers; ++l) {
        const LayerWeights& L = m->layers[l];
        kv_t* kvl = kv->pages + l * kv->layer_stride;
        rmsnorm(w.x, L.g_attn, w.xn, T, d.d_model, d.norm_eps, nullptr, nullptr, st);
        if (fuse_rope) {  // QKV GEMM with RoPE + q / paged-KV stores in its epilogue
            GemmProblem pq = lp(gp(w.xn, w.rows, L.wqkv, qkv_w, T, qkv_w, d.d_model, EPI_QKV_ROPE, false, nullptr, 0));
            pq.fx.pos = dev(tpos);
            pq.fx.slot = dev(tslot);
            pq.fx.page_table = kv->page_table;
            pq.fx.max_pages = kv->max_pages;
            pq.fx.page_tokens = B;
            pq.fx.rope_cs = m->rope_cs;
            pq.fx.q_out = w.q;
            pq.fx.kv_layer = kvl;
            pq.fx.page_stride = kv->page_stride;
            pq.fx.H = d.n_heads;
            pq.fx.Hkv = d.n_kv_heads;
            pq.fx.hd = d.head_dim;
            gemm_run(pq, st);
        } else {
            gemm_run(lp(gp(w.xn, w.rows, L.wqkv, qkv_w, T, qkv_w, d.d_model, EPI_STORE_F32, false, w.qkv, qkv_w)), st);
            rope_kv(w.qkv, w.q, kvl, dev(tpos), dev(tslot), kv->page_table, m->rope_cs, T, nullptr, d.n_heads,
                    d.n_kv_heads, d.head_dim, kv->max_pages, B, st);
        }
        if (Tp == 0) {
            // decode rows only (a token step through the prefill kernels): no prompt attention
        } else if (use_tc) {
            ta.layer_row0 = static_cast<int>(l * kv->layer_stride / d.head_dim);
            attn_prefill_tc(tm_q, kv->tm_kv, w.attn, ta, n_tiles128, d.head_dim, tc_persist, st);
        } else {
            attn_prefill(w.q, kvl, w.attn, aa, n_tiles, d.head_dim, st);
        }
        if (D > 0) {
            if (flat) {
                fa.layer_row0 = static_cast<int>(l * kv->layer_stride / d.head_dim);
                attn_decode_flat(kv->tm_kv, q_dec, attn_dec, fa, stream_sm_count(st), d.head_dim,
                                 d.n_heads / d.n_kv_heads, st);
            } else {
                attn_decode(q_dec, kvl, attn_dec, da, R, d.head_dim, st);
            }
        }
        gemm_run(lp(gp(w.attn, w.rows, L.wo, d.d_model, T, d.d_model, hdH, EPI_RESID, false, w.x, d.d_model)), st);
        rmsnorm(w.x, L.g_mlp, w.xn, T, d.d_model, d.norm_eps, nullptr, nullptr, st);
        gemm_run(lp(gp(w.xn, w.rows, L.wgu, 2 * d.ffn_dim, T, 2 * d.ffn_dim, d.d_model, EPI_SWIGLU, false, w.act,
                       d.ffn_dim)),
                 st);
        gemm_run(lp(gp(w.act, w.rows, L.wd, d.d_model, T, d.d_model, d.ffn_dim, EPI_RESID, false, w.x, d.d_model)), st);
    }
    // ---- last position of every prompt (+ every decode row) -> LM head + greedy token
    rmsnorm(w.x, m->g_final, w.xlast, NL, d.d_model, d.norm_eps, nullptr, dev(lastrow), st);
    lm_head(m, w, NL, nullptr, logits_out, st);
    finalize_tokens(w.keys, dev(sslot), dev(oidx), NL, nullptr, kv->last_token, kv->out_tokens, kv->max_out, st);
}

}  // namespace

void mixed_forward(sw_model* m, sw_kv* kv, const sw_batch& pre, const sw_batch& dec, cudaStream_t st,
                   float* logits_out) {
    int T = 0;
    for (int i = 0; i < pre.n; ++i) T += pre.n_tokens[i];
    if (pre.n < 0 || dec.n < 1) throw ConfigError("mixed step: needs at least one decode row");
    if (dec.n > kMaxDecodeRows) throw ContractViolation("mixed step: decode rows out of range");
    if (pre.n > kLmRowsMax) throw ConfigError("mixed step: at most 256 prompts per launch");
    if (T + dec.n > m->pre.rows)
        throw ConfigError("mixed step: prompt tokens + decode rows exceed one prefill launch (max_prefill_tokens=" +
                          std::to_string(m->pre.rows) + ")");
    if (!m->mix.meta) {
        ws_alloc(m->mix, m->desc, 1, true, 16);  // StepMeta + split-KV / flat partials + sum(x^2) scratch
        ring_init(m->mix_ring, 8, sizeof(StepMeta));
    }
    prefill_chunk(m, kv, pre, 0, pre.n, 0, 0, &dec, logits_out, st, false, 0);
}

}  // namespace sw

// ====================================================================== C-ABI
using namespace sw;

extern "C" int sw_model_create(const sw_model_desc* desc, int device, sw_model** out) {
    return guarded([&] {
        if (!desc || !out) throw ConfigError("sw_model_create: null argument");
        const sw_model_desc& d = *desc;
        if (d.n_layers < 1 || d.d_model % 64 || d.n_heads < 1 || d.n_kv_heads < 1 || d.n_heads % d.n_kv_heads ||
            (d.head_dim != 64 && d.head_dim != 128) || d.ffn_dim % 64 || d.vocab % 128 || d.vocab < 128)
            throw ConfigError("model: unsupported shape (d%64, hd in {64,128}, ffn%64, vocab%128, H%Hkv)");
        if (((d.n_heads + 2 * d.n_kv_heads) * d.head_dim) % 256 || d.d_model % 256 || (2 * d.ffn_dim) % 256)
            throw ConfigError("model: projection widths must be multiples of 256");
        if (d.max_prefill_tokens < 64 || d.max_decode_batch < 1 || d.max_decode_batch > kMaxDecodeRows)
            throw ConfigError("model: bad workspace sizes");
        SW_CUDA(cudaSetDevice(device));
        auto m = std::make_unique<sw_model>();
        m->desc = d;
        m->device = device;
        const int64_t D = d.d_model, V = d.vocab, F = d.ffn_dim, hd = d.head_dim;
        const int64_t qkv_w = (d.n_heads + 2 * d.n_kv_heads) * hd;
        // carve the weight arena
        std::vector<std::pair<std::string, int64_t>> plan;
        plan.push_back({"emb", V * D});
        if (!d.tied_embeddings) plan.push_back({"lm", V * D});
        plan.push_back({"g_final", D});
        for (int l = 0; l < d.n_layers; ++l) {
            const std::string p = "layer" + std::to_string(l) + ".";
            plan.push_back({p + "wqkv", qkv_w * D});
            plan.push_back({p + "wo", D * d.n_heads * hd});
            plan.push_back({p + "wgu", 2 * F * D});
            plan.push_back({p + "wd", D * F});
            plan.push_back({p + "g_attn", D});
            plan.push_back({p + "g_mlp", D});
        }
        size_t total = 0;
        for (auto& [n, e] : plan) total = align_up(total, 256) + static_cast<size_t>(e) * 2;
        m->weight_bytes = total;
        SW_CUDA(cudaMalloc(&m->weight_arena, total));
        size_t off = 0;
        for (auto& [n, e] : plan) {
            off = align_up(off, 256);
            m->tensors[n] = {static_cast<char*>(m->weight_arena) + off, e};
            off += static_cast<size_t>(e) * 2;
        }
        auto T = [&](const std::string& n) { return static_cast<__nv_bfloat16*>(m->tensors.at(n).first); };
        m->emb = T("emb");
        m->lm = d.tied_embeddings ? m->emb : T("lm");
        m->g_final = T("g_final");
        cudaStream_t st = nullptr;
        // synthetic weights: tensor k, element i of the LOGICAL [out, in] shape (oracle/model.py)
        const uint64_t seed = d.seed;
        init_tensor(m->emb, V, D, seed, 0, D, 0, 0, 0, st);
        fill_bf16(m->g_final, D, 1.0f, st);
        const int H = d.n_heads, Hk = d.n_kv_heads;
        for (int l = 0; l < d.n_layers; ++l) {
            const std::string p = "layer" + std::to_string(l) + ".";
            LayerWeights L{};
            L.wqkv = T(p + "wqkv");
            L.wo = T(p + "wo");
            L.wgu = T(p + "wgu");
            L.wd = T(p + "wd");
            L.g_attn = T(p + "g_attn");
            L.g_mlp = T(p + "g_mlp");
            const int k0 = 1 + 7 * l;
            init_tensor(L.wqkv, H * hd, D, seed, k0 + 0, D, 0, 0, 0, st);
            init_tensor(L.wqkv + H * hd * D, Hk * hd, D, seed, k0 + 1, D, 0, 0, 0, st);
            init_tensor(L.wqkv + (H + Hk) * hd * D, Hk * hd, D, seed, k0 + 2, D, 0, 0, 0, st);
            init_tensor(L.wo, D, H * hd, seed, k0 + 3, H * hd, 0, 0, 0, st);
            init_tensor(L.wgu, F, D, seed, k0 + 4, D, 64, 128, 0, st);   // gate rows -> [128j, 128j+64)
            init_tensor(L.wgu, F, D, seed, k0 + 5, D, 64, 128, 64, st);  // up rows   -> [128j+64, 128j+128)
            init_tensor(L.wd, D, F, seed, k0 + 6, F, 0, 0, 0, st);
            fill_bf16(L.g_attn, D, 1.0f, st);
            fill_bf16(L.g_mlp, D, 1.0f, st);
            m->layers.push_back(L);
        }
        if (!d.tied_embeddings) init_tensor(m->lm, V, D, seed, 1 + 7 * d.n_layers, D, 0, 0, 0, st);
        std::vector<float> inv(hd / 2);
        for (int i = 0; i < hd / 2; ++i)
            inv[i] = static_cast<float>(1.0 / std::pow(static_cast<double>(d.rope_theta), 2.0 * i / hd));
        m->inv_freq = dalloc<float>(hd / 2);
        SW_CUDA(cudaMemcpy(m->inv_freq, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
        m->rope_cs = dalloc<float2>(static_cast<size_t>(kMaxPositions) * (hd / 2));
        rope_table(m->inv_freq, m->rope_cs, kMaxPositions, static_cast<int>(hd / 2), st);
        ws_alloc(m->pre, d, d.max_prefill_tokens, false, 1);
        ws_alloc(m->dec[0], d, std::min(d.max_decode_batch, kMaxDecodeRows), true, 16);
        ring_init(m->pre_ring, 4, m->pre.pmeta_bytes);
        ring_init(m->dec_ring[0], 8, sizeof(StepMeta));
        m->scratch_u64 = dalloc<unsigned long long>(1);
        SW_CUDA(cudaDeviceSynchronize());
        *out = m.release();
    });
}

extern "C" int sw_model_destroy(sw_model* m) {
    return guarded([&] {
        if (!m) return;
        cudaDeviceSynchronize();
        for (auto& [k, g] : m->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        std::vector<Workspace*> all{&m->pre, &m->mix};
        for (auto& w : m->dec) all.push_back(&w);
        for (Workspace* w : all) {
            for (void* p : {(void*)w->x, (void*)w->xn, (void*)w->qkv, (void*)w->q, (void*)w->attn, (void*)w->act,
                            (void*)w->xlast, (void*)w->keys, (void*)w->meta, (void*)w->part_o, (void*)w->part_ml,
                            (void*)w->pmeta, (void*)w->splitk_ws, (void*)w->splitk_cnt, (void*)w->attn_cnt,
                            (void*)w->ss, (void*)w->flat_o, (void*)w->flat_ml})
                if (p) cudaFree(p);
        }
        std::vector<PinnedRing*> rings{&m->pre_ring, &m->mix_ring};
        for (auto& r : m->dec_ring) rings.push_back(&r);
        for (PinnedRing* r : rings) {
            for (void* p : r->slots) cudaFreeHost(p);
            for (cudaEvent_t e : r->done) cudaEventDestroy(e);
        }
        cudaFree(m->inv_freq);
        cudaFree(m->rope_cs);
        cudaFree(m->scratch_u64);
        cudaFree(m->weight_arena);
        delete m;
    });
}

extern "C" int sw_model_weight_checksum(sw_model* m, uint64_t* out) {
    return guarded([&] {
        SW_CUDA(cudaMemset(m->scratch_u64, 0, 8));
        checksum_bf16(m->weight_arena, static_cast<int64_t>(m->weight_bytes / 2), m->scratch_u64, nullptr);
        unsigned long long v = 0;
        SW_CUDA(cudaMemcpy(&v, m->scratch_u64, 8, cudaMemcpyDeviceToHost));
        *out = v;
    });
}

extern "C" int sw_model_tensor(sw_model* m, const char* name, void** ptr, int64_t* numel) {
    return guarded([&] {
        auto it = m->tensors.find(name);
        if (it == m->tensors.end()) throw ConfigError(std::string("model: no tensor '") + name + "'");
        *ptr = it->second.first;
        *numel = it->second.second;
    });
}

extern "C" int sw_kv_arena_create(sw_model* m, int64_t n_pages, int32_t n_slots, int32_t max_pages_per_slot,
                                  int32_t max_out_tokens, sw_kv** out) {
    return guarded([&] {
        if (!m || !out || n_pages < 1 || n_slots < 1 || max_pages_per_slot < 1 || max_out_tokens < 1)
            throw ConfigError("sw_kv_arena_create: bad arguments");
        if (static_cast<int64_t>(max_pages_per_slot) * 16 > kMaxPositions)
            throw ConfigError("sw_kv_arena_create: context longer than " + std::to_string(kMaxPositions) + " tokens");
        const sw_model_desc& d = m->desc;
        auto kv = std::make_unique<sw_kv>();
        kv->model = m;
        kv->n_pages = n_pages;
        kv->n_slots = n_slots;
        kv->max_pages = max_pages_per_slot;
        kv->max_out = max_out_tokens;
        kv->page_tokens = 16;
        kv->page_stride = 2LL * d.n_kv_heads * kv->page_tokens * d.head_dim;
        kv->layer_stride = kv->page_stride * n_pages;
        const size_t bytes = static_cast<size_t>(kv->layer_stride) * d.n_layers * 2;
        SW_CUDA(cudaMalloc(&kv->pages, bytes));
        // rows past a context inside its last page are read (and masked) by the
        // decode attention: keep them finite
        SW_CUDA(cudaMemset(kv->pages, 0, bytes));
        {
            const uint64_t rows = bytes / (2ull * d.head_dim);
            if (rows < (1ull << 31) && d.head_dim % 64 == 0) {
                kv->tm_kv = make_tmap_bf16(kv->pages, rows, d.head_dim, 16, /*fp16=*/true);
                kv->tm_kv_ok = true;
            }
        }
        kv->page_table = dalloc<int32_t>(static_cast<size_t>(n_slots) * max_pages_per_slot);
        SW_CUDA(cudaMemset(kv->page_table, 0, static_cast<size_t>(n_slots) * max_pages_per_slot * 4));
        kv->last_token = dalloc<int32_t>(n_slots);
        SW_CUDA(cudaMemset(kv->last_token, 0, static_cast<size_t>(n_slots) * 4));
        kv->out_tokens = dalloc<int32_t>(static_cast<size_t>(n_slots) * max_out_tokens);
        SW_CUDA(cudaMemset(kv->out_tokens, 0xff, static_cast<size_t>(n_slots) * max_out_tokens * 4));
        // split-KV: the kernel picks 1..16 splits per launch (grid x = 16)
        kv->chunk = 0;
        kv->max_splits = 16;
        *out = kv.release();
    });
}

extern "C" int sw_kv_arena_destroy(sw_kv* kv) {
    return guarded([&] {
        if (!kv) return;
        cudaDeviceSynchronize();
        for (auto it = kv->model->graphs.begin(); it != kv->model->graphs.end();) {
            if (std::get<0>(it->first) == kv) {
                if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
                it = kv->model->graphs.erase(it);
            } else {
                ++it;
            }
        }
        cudaFree(kv->pages);
        cudaFree(kv->page_table);
        cudaFree(kv->last_token);
        cudaFree(kv->out_tokens);
        delete kv;
    });
}

extern "C" int sw_kv_arena_views(sw_kv* kv, int32_t** page_table, int32_t** last_token, int32_t** out_tokens,
                                 void** pages) {
    return guarded([&] {
        if (page_table) *page_table = kv->page_table;
        if (last_token) *last_token = kv->last_token;
        if (out_tokens) *out_tokens = kv->out_tokens;
        if (pages) *pages = kv->pages;
    });
}

extern "C" int sw_prefill_enqueue(sw_model* m, sw_kv* kv, const sw_batch* b, void* stream) {
    return guarded([&] {
        if (!m || !kv || !b || !b->slots || !b->n_tokens || !b->tokens || !b->page_rows)
            throw ConfigError("sw_prefill_enqueue: null argument");
        prefill_forward(m, kv, *b, static_cast<cudaStream_t>(stream));
    });
}

extern "C" int sw_decode_enqueue(sw_model* m, sw_kv* kv, const sw_batch* b, void* stream) {
    return guarded([&] {
        if (!m || !kv || !b || !b->slots || !b->positions) throw ConfigError("sw_decode_enqueue: null argument");
        decode_forward(m, kv, *b, static_cast<cudaStream_t>(stream), /*use_graph=*/b->logits_out == nullptr);
    });
}

// ---- op level (kernel unit tests)
extern "C" int sw_op_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t epilogue,
                          void* stream) {
    return guarded([&] {
        // A = activations [M, K], B = weights [N, K]; swap-AB (+ split-K) when M <= 256
        const bool swap = M <= 256;
        static Workspace op_ws;  // split-K scratch for op-level calls
        if (!op_ws.splitk_ws) {
            op_ws.splitk_floats = static_cast<size_t>(kSplitTiles) * 256 * 128;
            op_ws.splitk_ws = dalloc<float>(op_ws.splitk_floats);
            op_ws.splitk_cnt = dalloc<unsigned>(kSplitCounters);
            SW_CUDA(cudaMemset(op_ws.splitk_cnt, 0, kSplitCounters * sizeof(unsigned)));
        }
        GemmProblem p = gp(A, M, B, N, M, N, K, epilogue, swap, C, epilogue == EPI_SWIGLU ? N / 2 : N, nullptr,
                           swap ? &op_ws : nullptr);
        gemm_run(p, static_cast<cudaStream_t>(stream));
    });
}

extern "C" int sw_op_rmsnorm(const float* x, const void* gain, void* y, int32_t rows, int32_t dim, float eps,
                             void* stream) {
    return guarded([&] {
        rmsnorm(x, static_cast<const __nv_bfloat16*>(gain), static_cast<__nv_bfloat16*>(y), rows, dim, eps, nullptr,
                nullptr, static_cast<cudaStream_t>(stream));
    });
}

extern "C" int sw_op_decode_attention(sw_model* m, sw_kv* kv, const sw_batch* b, void* stream) {
    return guarded([&] {
        if (!m || !kv || !b || !b->slots || !b->positions) throw ConfigError("sw_op_decode_attention: null argument");
        decode_attention_only(m, kv, *b, static_cast<cudaStream_t>(stream));
    });
}

extern "C" int sw_mixed_enqueue(sw_model* m, sw_kv* kv, const sw_batch* pre, const sw_batch* dec, void* stream) {
    return guarded([&] {
        if (!m || !kv || !pre || !dec || !pre->slots || !pre->n_tokens || !pre->tokens || !pre->page_rows ||
            !dec->slots || !dec->positions)
            throw ConfigError("sw_mixed_enqueue: null argument");
        mixed_forward(m, kv, *pre, *dec, static_cast<cudaStream_t>(stream), pre->logits_out);
    });
}

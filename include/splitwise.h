/*
 * splitwise.h -- C-ABI of the B200-native split-phase inference engine.
 *
 * Everything here is `extern "C"`, POD-only and exception-free: every call
 * returns an int status (SW_OK = 0, negative on error) and sw_last_error()
 * gives the message of the last failure on the calling thread.  Status codes
 * carry the reference's error taxonomy (splitsim/errors.hpp:9-30 mapped to
 * CLI exit codes in tools/splitsim.cpp:124-139): SW_ECONFIG (ConfigError /
 * ParseError, exit 2), SW_EIO (IoError, exit 3), SW_ECONTRACT
 * (ContractViolation, exit 4), SW_ECUDA (kernel/launch failure, reported as
 * a contract violation by the C++ executor).
 *
 * Two levels:
 *  1. Run level -- what the reference's run_config / run_simulation do
 *     (experiment.hpp:25-32, engine.hpp:497-500): a workload + policy spec in,
 *     an event log (same CSV as splitsim/event_log.hpp:113-261) + report out.
 *       sw_sim_run     virtual-clock backend (parity with the reference)
 *       sw_engine_run  real GPU backend (prefill and decode on B200)
 *  2. Kernel level -- the calls the GPU executor makes when it activates a
 *     task (replaces pricing a PhaseTask with make_prompt_task /
 *     make_token_step_task, gpu_model.hpp:154-189, by real forward passes):
 *       sw_model_create / sw_kv_arena_create / sw_prefill_enqueue /
 *       sw_decode_enqueue.  Stream-ordered; host arrays are staged by the call.
 */
#ifndef SPLITWISE_H
#define SPLITWISE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_OK 0
#define SW_ECONFIG (-2)
#define SW_EIO (-3)
#define SW_ECONTRACT (-4)
#define SW_ECUDA (-5)

typedef struct sw_model sw_model;
typedef struct sw_kv sw_kv;

/* Llama-style decoder shape (RMSNorm, RoPE, GQA attention, SwiGLU, greedy). */
typedef struct sw_model_desc {
    int32_t n_layers;
    int32_t d_model;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t head_dim;
    int32_t ffn_dim;
    int32_t vocab;
    int32_t tied_embeddings; /* LM head reuses the embedding table */
    float rope_theta;
    float norm_eps;
    uint64_t seed;            /* weights: SplitMix64 stream per tensor */
    int32_t max_prefill_tokens; /* prefill workspace, tokens per launch chunk */
    int32_t max_decode_batch;   /* decode workspace, rows per step */
} sw_model_desc;

/* One prefill (prompt) or decode (token step) launch over a set of requests.
 * All pointers are HOST pointers; the enqueue stages them to the device.
 *   prefill: row i covers prompt tokens [0, n_tokens[i]) of slot slots[i];
 *            tokens = concatenation of every row's prompt (sum n_tokens ints);
 *            page_rows = concatenation of every row's page-table prefix
 *            (ceil(n_tokens/page_tokens) ints each).
 *   decode:  row i feeds one token at position positions[i] of slot slots[i];
 *            tokens == NULL feeds the slot's last generated token (device
 *            resident, no host round trip); new_page[i] >= 0 installs that page
 *            id at page-table index positions[i]/page_tokens first.
 * Outputs: argmax token of each row -> device last_token[slot] and
 * out_tokens[slot][out_index[i]]; logits_out (device fp32 [n, vocab]) is
 * optional, for parity checks. */
typedef struct sw_batch {
    int32_t n;
    const int32_t* slots;
    const int32_t* n_tokens;  /* prefill */
    const int32_t* positions; /* decode: each row's position; prefill (may be NULL): each prompt chunk's
                                 first position, a multiple of 128, earlier positions already in its pages */
    const int32_t* tokens;
    const int32_t* page_rows; /* prefill */
    const int32_t* new_page;  /* decode, may be NULL */
    const int32_t* out_index; /* where the argmax lands in out_tokens[slot][] */
    float* logits_out;        /* device, may be NULL */
} sw_batch;

const char* sw_last_error(void);
void sw_free(void* p);
/* Kernels launched by this library so far (graph replays count their nodes). */
unsigned long long sw_launch_count(void);
/* Host->device and device->host bytes moved by the run path so far. */
void sw_transfer_bytes(unsigned long long* h2d, unsigned long long* d2h);

/* ---- run level ---- */
/* spec: `key=value;...` (see csrc/host/spec.hpp).  *out receives a malloc'd
 * text: the event-log CSV, then `#report k=v;...`, then `#pages` lines. */
int sw_sim_run(const char* spec, char** out);
int sw_engine_run(sw_model* model, sw_kv* kv, const char* spec, char** out);
/* Spec keys `output_dir=<dir>;emit_event_log=1` make both runs write the
 * reference's experiment files there (splitsim/experiment.hpp:194-212
 * write_experiment: report.json, requests.csv, timeseries.csv, events.csv).
 * sw_replay: rebuild the report of a written events.csv, write
 * replay_report.json next to it (experiment.hpp:290-296 replay_file +
 * tools/splitsim.cpp:73-85), *out = the `#report` text. */
int sw_replay(const char* events_path, char** out);

/* ---- kernel level ---- */
int sw_model_create(const sw_model_desc* desc, int device, sw_model** out);
int sw_model_destroy(sw_model* model);
int sw_model_weight_checksum(sw_model* model, uint64_t* out); /* parity of generated weights */
int sw_model_tensor(sw_model* model, const char* name, void** dev_ptr, int64_t* numel);

int sw_kv_arena_create(sw_model* model, int64_t n_pages, int32_t n_slots, int32_t max_pages_per_slot,
                       int32_t max_out_tokens, sw_kv** out);
int sw_kv_arena_destroy(sw_kv* kv);
/* KV capacity of the device in pages (the reference's derive_kv_capacity,
 * splitsim/config.hpp:66-79, with budget = cudaMemGetInfo free bytes -
 * reserve_bytes; one page = 16 tokens x 2 (K,V) x n_layers x n_kv_heads x
 * head_dim fp16 values, 2 MiB for Llama-3-8B).  Call after sw_model_create so
 * the weights are already resident. */
int sw_kv_capacity_pages(const sw_model_desc* desc, int device, int64_t reserve_bytes, int64_t* out);
/* Device arrays of the arena (page table int32 [n_slots][max_pages_per_slot],
 * last_token int32 [n_slots], out_tokens int32 [n_slots][max_out_tokens],
 * pages bf16 [n_layers][n_pages][2][n_kv_heads][page_tokens][head_dim]). */
int sw_kv_arena_views(sw_kv* kv, int32_t** page_table, int32_t** last_token, int32_t** out_tokens, void** pages);

/* One decode step's attention alone (every layer, the kernel the step would pick) over the batch's
 * paged contexts -- the timing probe bench.py uses for the roofline of the dominant decode kernel.
 * It uses decode lane 0's workspace: not concurrent with sw_decode_enqueue on the same model. */
int sw_op_decode_attention(sw_model* model, sw_kv* kv, const sw_batch* batch, void* stream);
int sw_prefill_enqueue(sw_model* model, sw_kv* kv, const sw_batch* batch, void* stream);
/* The co-scheduler's SM partition (green contexts, cached per device): a
 * decode stream on `decode_sms` SMs (rounded to the driver's granularity) and
 * a prefill stream on the rest; kernels enqueued on them stay on their SMs. */
int sw_sm_partition(int device, int decode_sms, void** decode_stream, void** prefill_stream, int* decode_sms_out,
                    int* prefill_sms_out);
int sw_decode_enqueue(sw_model* model, sw_kv* kv, const sw_batch* batch, void* stream);
/* One fused mixed step -- the split-phase co-execution of a prompt chunk and a
 * token step (MixedBatching's "one prompt and one step in flight together"):
 * the decode rows of `decode` (sw_decode_enqueue semantics) ride in the
 * prefill pass of `prefill` (sw_prefill_enqueue semantics), so each projection
 * GEMM streams its weights once for both phases.  All prompts and decode rows
 * must fit one launch (prompt tokens + rows <= max_prefill_tokens, prompts +
 * rows <= 256).  prefill->logits_out (optional) receives the prompts' last-
 * position logits followed by the decode rows'. */
int sw_mixed_enqueue(sw_model* model, sw_kv* kv, const sw_batch* prefill, const sw_batch* decode, void* stream);

/* ---- op level (kernel unit tests; device pointers, stream-ordered) ---- */
/* C[M,N] (+)= A[M,K] . B[N,K]^T, bf16 in, fp32 accumulate.
 * epilogue: 0 store bf16 C; 1 add into fp32 C (residual); 2 SwiGLU over
 * [gate 64 | up 64] column blocks -> bf16 C[M, N/2]. */
int sw_op_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t epilogue,
               void* stream);
int sw_op_rmsnorm(const float* x, const void* gain, void* y_bf16, int32_t rows, int32_t dim, float eps,
                  void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPLITWISE_H */

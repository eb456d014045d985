// GPU executor: the engine side of the reference contract (executor.hpp)
// driven by real prefill/decode forward passes on a B200 instead of the
// virtual clock (replaces splitsim::Engine::run, engine.hpp:101-172).
//
// One host thread runs the reference loop on device time:
//   poll    cudaEventQuery on every in-flight launch's end event;
//           arrivals are due when wall time since run start >= arrival_s;
//   drain   due arrivals and completed launches in time order (arrivals
//           first on ties, completions in activation order), applying the
//           exact completion semantics of the core (KV growth, finish, free);
//   pass    one scheduler pass; every activated task is enqueued as real
//           work -- a prompt task = prefill_forward over its prompts, a token
//           step = decode_forward over its running batch.
// Split phase: prompts go to the prefill stream, token steps to a
// higher-priority decode stream, so the compute-bound and HBM-bound phases
// overlap on the SMs and share the one paged KV arena (the handoff is a
// scheduler list append, no data moves).  Serial mode puts both on one
// stream: the same task stream, one kernel sequence at a time.
// Tasks activated in the same pass with the same kind are coalesced into one
// launch (one weight stream for several lanes' token steps).
// Timestamps: TaskStart = device time the launch began (event before its
// first kernel), TaskComplete = device time of its end event, both relative
// to an event recorded at run start; arrivals carry their nominal time.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/splitwise_engine.hpp"
#include "../host/capi_util.hpp"
#include "../host/executor.hpp"
#include "../host/report.hpp"
#include "../host/run_text.hpp"
#include "../host/spec.hpp"
#include "../kernels/common.cuh"
#include "model.hpp"
#include "../host/experiment_files.hpp"
#include "partition.hpp"

namespace sw {

// Algorithmic work of the real forward passes.
struct ModelWork {
    double n_mm = 0, d = 0, V = 0, L = 0, H = 0, hd = 0, kv_tok = 0;
    explicit ModelWork(const sw_model_desc& m) {
        d = m.d_model;
        V = m.vocab;
        L = m.n_layers;
        H = m.n_heads;
        hd = m.head_dim;
        const double qkv = (m.n_heads + 2.0 * m.n_kv_heads) * m.head_dim;
        n_mm = L * (d * qkv + m.n_heads * m.head_dim * d + 3.0 * d * m.ffn_dim);
        kv_tok = 2.0 * L * m.n_kv_heads * m.head_dim * 2.0;
    }
    double weight_bytes() const { return 2.0 * (n_mm + d * V); }
    double prompt_flops(double S) const { return 2.0 * n_mm * S + 2.0 * L * H * hd * S * (S + 1.0) + 2.0 * d * V; }
    double step_bytes(double b, double sum_ctx) const { return weight_bytes() + 2.0 * d * b + sum_ctx * kv_tok + b * kv_tok; }
    double step_flops(double b, double sum_ctx) const { return b * 2.0 * (n_mm + d * V) + 4.0 * L * H * hd * sum_ctx; }
};

class GpuExecutor final : public ExecutorCore {
public:
    GpuExecutor(const SimulationInputs& in, Scheduler& sched, sw_model* m, sw_kv* kv, const GpuOptions& opt)
        : ExecutorCore(in, sched), m_(m), kv_(kv), opt_(opt), work_(m->desc) {
        if (in_.discipline.mode == SharingDiscipline::Mode::TimeSliced)
            throw ConfigError("discipline.mode: time_sliced is not a GPU mode");
        if (static_cast<long long>(entries_.size()) > kv_->n_slots)
            throw ConfigError("engine: more requests than KV arena slots");
        if (pages_.n_pages() > kv_->n_pages) throw ConfigError("engine: kv_capacity_blocks exceeds the KV arena");
        int max_out = 0, max_ctx = 0;
        for (const Entry& e : entries_) {
            max_out = std::max(max_out, e.req.output_tokens);
            max_ctx = std::max(max_ctx, e.req.input_tokens + e.req.output_tokens);
        }
        if (max_out + 1 > kv_->max_out) throw ConfigError("engine: output longer than the arena's token buffer");
        if ((max_ctx + kv_->page_tokens - 1) / kv_->page_tokens > kv_->max_pages)
            throw ConfigError("engine: context longer than the arena's page-table row");
        for (std::size_t i = 0; i < entries_.size(); ++i) slot_of_[entries_[i].req.id] = static_cast<int>(i);
        const int lanes = opt_.split ? std::max(1, std::min(opt_.decode_lanes, sw_model::kMaxDecodeLanes)) : 1;
        if (opt_.split && opt_.decode_sms > 0) {
            // co-scheduler: decode and prefill on disjoint SM groups (green contexts, cached per model device)
            const SmPartition& P = sm_partition(m_->device, opt_.decode_sms, lanes);
            s_prefill_ = P.prefill;
            s_decode_ = P.decode;
            part_ = &P;
            own_streams_ = false;
            // prompts launched while no request is generating take the whole GPU, and so do
            // token steps launched while no prompt is in flight (the partition only pays
            // while both phases run: profiles/r01c/overlap_1b.txt)
            int lo, hi;
            SW_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            SW_CUDA(cudaStreamCreateWithPriority(&s_prefill_full_, cudaStreamNonBlocking, lo));
            for (int i = 0; i < lanes; ++i) {
                cudaStream_t sf;
                SW_CUDA(cudaStreamCreateWithPriority(&sf, cudaStreamNonBlocking, hi));
                s_decode_full_.push_back(sf);
            }
            return;
        }
        int lo, hi;
        SW_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        // engine.prefill_priority=1 (default): the prefill stream outranks the decode streams (a
        // prompt that shares the GPU with token steps finishes first -- the lanes' steps then merge
        // sooner, and back-to-back steps cannot starve prompts); =0: token steps first
        const int p_pre = opt_.prefill_priority ? hi : lo, p_dec = opt_.prefill_priority ? lo : hi;
        SW_CUDA(cudaStreamCreateWithPriority(&s_prefill_, cudaStreamNonBlocking, p_pre));
        for (int i = 0; i < lanes; ++i) {
            cudaStream_t s = s_prefill_;
            if (opt_.split) SW_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, p_dec));
            s_decode_.push_back(s);
        }
    }

    ~GpuExecutor() override {
        cudaStreamSynchronize(s_prefill_);
        for (cudaStream_t s : s_decode_) cudaStreamSynchronize(s);
        for (cudaEvent_t e : events_) cudaEventDestroy(e);
        if (s_prefill_full_) {
            cudaStreamSynchronize(s_prefill_full_);
            cudaStreamDestroy(s_prefill_full_);
        }
        for (cudaStream_t s : s_decode_full_) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
        if (!own_streams_) return;
        for (cudaStream_t s : s_decode_)
            if (s != s_prefill_) cudaStreamDestroy(s);
        cudaStreamDestroy(s_prefill_);
    }

    EventLog run() {
        using clk = std::chrono::steady_clock;
        t0_ = new_event();
        SW_CUDA(cudaEventRecord(events_[t0_], s_prefill_));
        SW_CUDA(cudaEventSynchronize(events_[t0_]));
        const auto wall0 = clk::now();
        seq_ = static_cast<long long>(entries_.size());
        std::size_t next_arrival = 0;
        bool first = true;
        for (;;) {
            const double now = std::chrono::duration<double>(clk::now() - wall0).count();
            // ---- poll
            struct Ev {
                double t;
                int kind;  // 0 arrival, 1 completion
                long long order;
                std::size_t ref;
            };
            std::vector<Ev> evs;
            while (next_arrival < entries_.size() && entries_[next_arrival].req.arrival_s <= now) {
                evs.push_back({entries_[next_arrival].req.arrival_s, 0, static_cast<long long>(next_arrival), next_arrival});
                ++next_arrival;
            }
            for (std::size_t i = 0; i < launches_.size(); ++i) {
                Launch& L = launches_[i];
                if (L.done) continue;
                const cudaError_t q = cudaEventQuery(events_[L.end_ev]);
                if (q == cudaErrorNotReady) continue;
                SW_CUDA(q);
                L.done = true;
                L.t_end = elapsed(L.end_ev);
                evs.push_back({L.t_end, 1, L.first_seq, i});
            }
            std::stable_sort(evs.begin(), evs.end(), [](const Ev& a, const Ev& b) {
                if (a.t != b.t) return a.t < b.t;
                if (a.kind != b.kind) return a.kind < b.kind;
                return a.order < b.order;
            });
            for (const Ev& e : evs) {
                clock_ = std::max(clock_, e.t);
                if (e.kind == 0) {
                    log_arrival(entries_[e.ref], {e.t});
                } else {
                    for (long long sq : launches_[e.ref].task_seqs) {
                        std::size_t idx = 0;
                        while (idx < active_.size() && active_[idx].seq != sq) ++idx;
                        if (idx == active_.size()) throw ContractViolation("gpu executor: lost task");
                        complete(idx, {e.t});
                    }
                }
            }
            if (!evs.empty() || first) {
                first = false;
                schedule_pass();
            }
            flush_steps();
            const bool inflight = !pending_steps_.empty() || !jobs_.empty() ||
                                  std::any_of(launches_.begin(), launches_.end(), [](const Launch& l) { return !l.done; });
            if (!inflight && active_.empty() && next_arrival >= entries_.size()) break;
            if (!inflight && active_.empty() && evs.empty()) {
                // idle until the next arrival
                const double wait = entries_[next_arrival].req.arrival_s - now;
                if (wait > 2e-4) std::this_thread::sleep_for(std::chrono::duration<double>(wait - 1e-4));
            } else if (evs.empty()) {
                std::this_thread::yield();
            }
            if (++polls_ > 2'000'000'000ULL) throw ContractViolation("gpu executor: livelock guard");
        }
        check_all_finished();
        double t_end = clock_;
        LogRecord end;
        end.kind = LogKind::RunEnd;
        append(end, {t_end});
        clock_skew_ = finalize_times([&](int ev) { return elapsed(ev); }, /*align_device_clock=*/true);
        // RunEnd must stay last: after sorting it is (all stamps <= clock_).
        return log_;
    }

    // Generated tokens, device page-table rows and launch statistics of the run.
    void collect(RunOutputs& o) const {
        // generated tokens per request: x_1..x_out (device out_tokens[slot][0..out))
        std::vector<int32_t> host(static_cast<size_t>(kv_->n_slots) * kv_->max_out);
        SW_CUDA(cudaMemcpy(host.data(), kv_->out_tokens, host.size() * 4, cudaMemcpyDeviceToHost));
        std::vector<int32_t> table(static_cast<size_t>(kv_->n_slots) * kv_->max_pages);
        SW_CUDA(cudaMemcpy(table.data(), kv_->page_table, table.size() * 4, cudaMemcpyDeviceToHost));
        count_transfer(0, (host.size() + table.size()) * 4);
        for (const Entry& e : entries_) {
            const std::size_t slot = static_cast<std::size_t>(slot_of_.at(e.req.id));
            const int32_t* t = host.data() + slot * static_cast<std::size_t>(kv_->max_out);
            o.tokens[e.req.id].assign(t, t + e.req.output_tokens);
            const auto it = pages_.final_rows().find(e.req.id);
            const std::size_t np = it == pages_.final_rows().end() ? 0 : it->second.size();
            const int32_t* r = table.data() + slot * static_cast<std::size_t>(kv_->max_pages);
            o.page_rows[e.req.id].assign(r, r + np);
        }
        char buf[512];
        std::snprintf(buf, sizeof buf,
                      "#gpu launches=%zu;prefill_launches=%d;decode_launches=%d;split=%d;coalesce=%d;align=%d;decode_lanes=%zu;"
                      "decode_sms=%d;prefill_sms=%d;prefill_full_gpu=%d;decode_full_gpu=%d;prefill_lean=%d;prefill_yield=%d;"
                      "fuse=%d;mixed_launches=%d;chunk_tokens=%d;clock_skew_s=%.9g\n",
                      launches_.size(), n_prefill_, n_decode_, opt_.split ? 1 : 0, opt_.coalesce ? 1 : 0,
                      aligning() ? 1 : 0, s_decode_.size(), part_ ? part_->decode_sms : 0, part_ ? part_->prefill_sms : 0, n_prefill_full_,
                      n_decode_full_, n_prefill_lean_, n_prefill_yield_, fusing() ? 1 : 0, n_mixed_, opt_.chunk_tokens,
                      clock_skew_);
        o.diagnostics = buf;
        o.pages = pages_;
    }

protected:
    PhaseTask price(const TaskRequest& tr, const std::vector<Request>& prompt_batch) override {
        PhaseTask t;
        t.kind = tr.kind;
        t.instance_id = tr.instance_id;
        t.batch = tr.batch;
        check_batch(t.batch);
        if (tr.kind == TaskKind::Prompt) {
            double flops = 0, toks = 0;
            for (const Request& r : prompt_batch) {
                flops += work_.prompt_flops(r.input_tokens);
                toks += r.input_tokens;
            }
            t.compute_demand = flops;
            t.mem_demand = work_.weight_bytes() + toks * work_.kv_tok;
        } else {
            double ctx = 0;
            for (int rid : tr.batch) {
                const Entry& e = entry(rid);
                ctx += e.req.input_tokens + e.generated;  // keys attended (incl. the fed token)
            }
            const double b = static_cast<double>(tr.batch.size());
            t.compute_demand = work_.step_flops(b, ctx);
            t.mem_demand = work_.step_bytes(b, ctx - b);
        }
        t.duration_alone_s = std::max(t.compute_demand / opt_.peak_flops, t.mem_demand / opt_.peak_bytes);
        return t;
    }

private:
    struct Launch {
        TaskKind kind;
        int lane = 0;
        int start_ev = -1, end_ev = -1;
        std::vector<std::pair<int, int>> merged_evs;  // (start, end) events of launches merged into this one
        std::vector<long long> task_seqs;
        long long first_seq = 0;
        bool done = false;
        double t_end = 0;
    };

    int new_event() {
        cudaEvent_t e;
        SW_CUDA(cudaEventCreate(&e));
        events_.push_back(e);
        return static_cast<int>(events_.size()) - 1;
    }

    double elapsed(int ev) const {
        float ms = 0.f;
        SW_CUDA(cudaEventElapsedTime(&ms, events_[t0_], events_[ev]));
        return static_cast<double>(ms) * 1e-3;
    }

    void schedule_pass() {
        const std::vector<TaskRequest> trs = pass_tasks();
        if (trs.empty()) return;
        // group: coalesced -> one launch per kind; else one per task
        std::vector<Launch> group;
        int prompt_launch = -1;
        std::vector<std::pair<int, std::size_t>> placement;  // (launch idx in group, active idx)
        std::map<int, int> step_launch_of_lane;
        for (const TaskRequest& tr : trs) {
            int gi;
            const int lane = static_cast<int>(tr.instance_id % static_cast<int>(s_decode_.size()));
            int& slot = tr.kind == TaskKind::Prompt ? prompt_launch
                                                    : (step_launch_of_lane.count(lane) ? step_launch_of_lane[lane]
                                                                                       : (step_launch_of_lane[lane] = -1));
            if (opt_.coalesce && slot >= 0) {
                gi = slot;
            } else {
                Launch L;
                L.kind = tr.kind;
                L.lane = lane;
                L.start_ev = new_event();
                L.end_ev = new_event();
                group.push_back(L);
                gi = static_cast<int>(group.size()) - 1;
                slot = gi;
            }
            const std::size_t ai = activate(tr, {0.0, group[static_cast<std::size_t>(gi)].start_ev});
            group[static_cast<std::size_t>(gi)].task_seqs.push_back(active_[ai].seq);
        }
        for (Launch& L : group) {
            L.first_seq = L.task_seqs.front();
            if (aligning() && L.kind == TaskKind::TokenStep) {
                pending_steps_.push_back(L);
                continue;
            }
            if (fusing() && L.kind == TaskKind::Prompt) {
                fuse_add_prompt(L);
                continue;
            }
            enqueue(L);
            launches_.push_back(L);
        }
        flush_steps();
    }

    // token steps of several lanes requested while one is in flight wait and run as one merged
    // launch -- in split mode and (round 2) in the serial arm too, so "serial" is the same task
    // stream on one stream, not a stream that re-reads the weights once per lane
    bool aligning() const { return opt_.align || (opt_.split && opt_.fuse); }
    bool fusing() const { return opt_.split && opt_.fuse; }

    // decode work exists: a step in flight or waiting, or a request past its prompt
    bool decode_active() const {
        if (decode_inflight() || !pending_steps_.empty()) return true;
        return std::any_of(entries_.begin(), entries_.end(),
                           [](const Entry& e) { return e.req.state == RequestState::Generating; });
    }

    bool prompt_inflight() const {
        return std::any_of(launches_.begin(), launches_.end(),
                           [](const Launch& l) { return !l.done && l.kind == TaskKind::Prompt; });
    }

    bool decode_inflight() const {
        return std::any_of(launches_.begin(), launches_.end(),
                           [](const Launch& l) { return !l.done && l.kind == TaskKind::TokenStep; });
    }

    // Aligned token steps: once no step is in flight, every waiting step runs as
    // one merged launch on decode lane 0 (their TaskStart/TaskComplete events
    // are all recorded around it).
    void flush_steps() {
        if (fusing()) {
            fuse_dispatch();
            return;
        }
        if (pending_steps_.empty() || decode_inflight()) return;
        Launch M = pending_steps_.front();
        M.lane = 0;
        for (std::size_t i = 1; i < pending_steps_.size(); ++i) {
            const Launch& o = pending_steps_[i];
            M.task_seqs.insert(M.task_seqs.end(), o.task_seqs.begin(), o.task_seqs.end());
            M.merged_evs.push_back({o.start_ev, o.end_ev});
        }
        pending_steps_.clear();
        enqueue(M);
        launches_.push_back(M);
    }

    // Host staging of one launch's batch (kept alive until the enqueue returns:
    // the forward passes stage host arrays into pinned memory themselves).
    struct BatchBuf {
        std::vector<int32_t> slots, ntok, pos, newp, oidx, toks, prow;
        sw_batch b{};
    };

    std::vector<int> rids_of(const std::vector<long long>& seqs) const {
        std::vector<int> rids;
        for (long long sq : seqs) {
            const Active* a = nullptr;
            for (const Active& x : active_)
                if (x.seq == sq) a = &x;
            if (!a) throw ContractViolation("gpu executor: enqueue of unknown task");
            rids.insert(rids.end(), a->task.batch.begin(), a->task.batch.end());
        }
        return rids;
    }

    // Prompt tokens [begin, end) a prompt task in flight covers for request rid: the whole prompt, or
    // one chunk of it (policy chunked_prefill).
    std::pair<int, int> chunk_range(int rid) const {
        for (const Active& a : active_) {
            if (a.task.kind != TaskKind::Prompt || a.task.chunk_end.empty()) continue;
            for (std::size_t i = 0; i < a.task.batch.size(); ++i)
                if (a.task.batch[i] == rid) return {a.task.chunk_begin[i], a.task.chunk_end[i]};
        }
        return {0, entry(rid).req.input_tokens};
    }

    void build_prompt(const std::vector<int>& rids, BatchBuf& B) const {
        const int n = static_cast<int>(rids.size());
        B.slots.resize(n);
        B.ntok.resize(n);
        B.pos.assign(n, 0);
        B.oidx.assign(n, 0);
        bool chunked = false;
        for (int i = 0; i < n; ++i) {
            const Entry& e = entry(rids[i]);
            const auto [b0, b1] = chunk_range(rids[i]);
            B.slots[i] = slot_of_.at(rids[i]);
            B.ntok[i] = b1 - b0;
            B.pos[i] = b0;
            chunked |= b0 > 0;
            // only a prompt's last chunk produces its first token
            B.oidx[i] = b1 == e.req.input_tokens ? 0 : -1;
            for (int j = b0; j < b1; ++j) B.toks.push_back(prompt_token(m_->desc.seed, e.req.id, j, m_->desc.vocab));
            const std::vector<int>& row = pages_.row(rids[i]);
            const int need = (b1 + kv_->page_tokens - 1) / kv_->page_tokens;
            for (int j = 0; j < need; ++j) B.prow.push_back(row.at(static_cast<std::size_t>(j)));
        }
        B.b.n = n;
        B.b.slots = B.slots.data();
        B.b.n_tokens = B.ntok.data();
        B.b.positions = chunked ? B.pos.data() : nullptr;
        B.b.tokens = B.toks.data();
        B.b.page_rows = B.prow.data();
        B.b.out_index = B.oidx.data();
    }

    void build_step(const std::vector<int>& rids, BatchBuf& B) const {
        const int n = static_cast<int>(rids.size());
        B.slots.resize(n);
        B.pos.resize(n);
        B.newp.resize(n);
        B.oidx.resize(n);
        for (int i = 0; i < n; ++i) {
            const Entry& e = entry(rids[i]);
            B.slots[i] = slot_of_.at(rids[i]);
            B.pos[i] = e.req.input_tokens + e.generated;  // position of the fed token x_g
            const int pidx = B.pos[i] / kv_->page_tokens;
            B.newp[i] = B.pos[i] % kv_->page_tokens == 0 ? pages_.row(rids[i]).at(static_cast<std::size_t>(pidx)) : -1;
            B.oidx[i] = e.generated + 1;  // x_{g+1}
        }
        B.b.n = n;
        B.b.slots = B.slots.data();
        B.b.positions = B.pos.data();
        B.b.new_page = B.newp.data();
        B.b.out_index = B.oidx.data();
    }

    void enqueue(const Launch& L) {
        const std::vector<int> rids = rids_of(L.task_seqs);
        BatchBuf B;
        if (L.kind == TaskKind::Prompt) {
            build_prompt(rids, B);
            // partition mode: the prefill group's SMs only while decode work exists, else the whole GPU
            const bool active = decode_active();
            cudaStream_t ps = s_prefill_full_ && !active ? s_prefill_full_ : s_prefill_;
            if (ps == s_prefill_full_) ++n_prefill_full_;
            const bool lean = opt_.split && opt_.lean_prefill && active;
            n_prefill_lean_ += lean ? 1 : 0;
            SW_CUDA(cudaEventRecord(events_[L.start_ev], ps));
            const int yield = opt_.split && active ? opt_.prefill_yield : 0;
            n_prefill_yield_ += yield > 0 ? 1 : 0;
            prefill_forward(m_, kv_, B.b, ps, lean, yield);
            SW_CUDA(cudaEventRecord(events_[L.end_ev], ps));
            ++n_prefill_;
        } else {
            build_step(rids, B);
            cudaStream_t ds = s_decode_[static_cast<std::size_t>(L.lane)];
            if (!s_decode_full_.empty() && !prompt_inflight()) {  // partition mode, decode alone: whole GPU
                ds = s_decode_full_[static_cast<std::size_t>(L.lane)];
                ++n_decode_full_;
            }
            SW_CUDA(cudaEventRecord(events_[L.start_ev], ds));
            for (const auto& [se, ee] : L.merged_evs) SW_CUDA(cudaEventRecord(events_[se], ds));
            decode_forward(m_, kv_, B.b, ds, opt_.graphs, L.lane, static_cast<int>(s_decode_.size()));
            SW_CUDA(cudaEventRecord(events_[L.end_ev], ds));
            for (const auto& [se, ee] : L.merged_evs) SW_CUDA(cudaEventRecord(events_[ee], ds));
            ++n_decode_;
        }
    }

    // ---- fused mixed steps (engine.fuse=1: chunked prefill with the
    // token step riding in each chunk).  A prompt task runs as chunks of whole prompts
    // (<= engine.chunk_tokens tokens); while it is in flight, every token step the
    // scheduler requests is merged into the next chunk's launch (mixed_forward: one
    // weight stream for both phases).  Launches go out one at a time on one stream, so
    // the step that completes with a chunk can be followed by its successor in the next.
    struct PromptJob {
        Launch L;  // the prompt task(s): start_ev recorded at the first chunk, end_ev at the last
        std::vector<std::vector<int>> chunks;
        std::size_t next = 0;
    };

    void fuse_add_prompt(const Launch& L) {
        PromptJob J;
        J.L = L;
        const std::vector<int> rids = rids_of(L.task_seqs);
        const int cap = std::max(1, std::min(opt_.chunk_tokens > 0 ? opt_.chunk_tokens : (1 << 30),
                                             m_->pre.rows - kMaxDecodeRows));
        std::vector<int> cur;
        int tok = 0;
        for (int rid : rids) {
            const auto [b0, b1] = chunk_range(rid);  // chunked_prefill tasks: this task's share of the prompt
            const int n = b1 - b0;
            if (!cur.empty() && (tok + n > cap || cur.size() >= 256)) {
                J.chunks.push_back(cur);
                cur.clear();
                tok = 0;
            }
            cur.push_back(rid);
            tok += n;
        }
        if (!cur.empty()) J.chunks.push_back(cur);
        jobs_.push_back(std::move(J));
    }

    bool fused_busy() const {
        return std::any_of(launches_.begin(), launches_.end(), [](const Launch& l) { return !l.done; });
    }

    void fuse_dispatch() {
        if (fused_busy()) return;
        PromptJob* J = jobs_.empty() ? nullptr : &jobs_.front();
        if (!J && pending_steps_.empty()) return;
        cudaStream_t st = s_prefill_;
        BatchBuf P, D;
        std::vector<int> chunk;
        bool first_chunk = false, last_chunk = false;
        int chunk_tok = 0;
        if (J) {
            chunk = J->chunks[J->next];
            first_chunk = J->next == 0;
            last_chunk = J->next + 1 == J->chunks.size();
            build_prompt(chunk, P);
            for (int v : P.ntok) chunk_tok += v;
        }
        // the waiting token steps, merged (one decode row set)
        Launch M;
        bool step = false;
        if (!pending_steps_.empty()) {
            M = pending_steps_.front();
            M.lane = 0;
            for (std::size_t i = 1; i < pending_steps_.size(); ++i) {
                const Launch& o = pending_steps_[i];
                M.task_seqs.insert(M.task_seqs.end(), o.task_seqs.begin(), o.task_seqs.end());
                M.merged_evs.push_back({o.start_ev, o.end_ev});
            }
            build_step(rids_of(M.task_seqs), D);
            // fuse only when the rows fit one prefill launch
            step = !J || chunk_tok + D.b.n <= m_->pre.rows;
            if (step) pending_steps_.clear();
        }
        // ---- launch start events
        Launch C;  // the chunk's in-flight record (carries the prompt task only on its last chunk)
        if (J) {
            C.kind = TaskKind::Prompt;
            C.start_ev = first_chunk ? J->L.start_ev : new_event();
            C.end_ev = last_chunk ? J->L.end_ev : new_event();
            if (last_chunk) C.task_seqs = J->L.task_seqs;
            C.first_seq = J->L.first_seq;
            SW_CUDA(cudaEventRecord(events_[C.start_ev], st));
        }
        if (step) {
            SW_CUDA(cudaEventRecord(events_[M.start_ev], st));
            for (const auto& [se, ee] : M.merged_evs) SW_CUDA(cudaEventRecord(events_[se], st));
        }
        // ---- the work
        if (J && step) {
            mixed_forward(m_, kv_, P.b, D.b, st);
            ++n_mixed_;
        } else if (J) {
            prefill_forward(m_, kv_, P.b, st);
            ++n_prefill_;
        } else {
            decode_forward(m_, kv_, D.b, st, opt_.graphs, 0, 1);
            ++n_decode_;
        }
        // ---- end events, in-flight records
        if (step) {
            SW_CUDA(cudaEventRecord(events_[M.end_ev], st));
            for (const auto& [se, ee] : M.merged_evs) SW_CUDA(cudaEventRecord(events_[ee], st));
            launches_.push_back(M);
        }
        if (J) {
            SW_CUDA(cudaEventRecord(events_[C.end_ev], st));
            launches_.push_back(C);
            if (++J->next == J->chunks.size()) jobs_.pop_front();
        }
    }

    sw_model* m_;
    sw_kv* kv_;
    GpuOptions opt_;
    ModelWork work_;
    cudaStream_t s_prefill_ = nullptr;
    std::vector<cudaStream_t> s_decode_;
    const SmPartition* part_ = nullptr;  // green-context partition (split mode, engine.decode_sms > 0)
    cudaStream_t s_prefill_full_ = nullptr;  // partition mode: whole-GPU prefill stream
    std::vector<cudaStream_t> s_decode_full_;  // partition mode: whole-GPU decode streams (per lane)
    int n_decode_full_ = 0;
    int n_prefill_full_ = 0;
    int n_prefill_lean_ = 0;
    int n_prefill_yield_ = 0;
    bool own_streams_ = true;
    std::vector<cudaEvent_t> events_;
    int t0_ = -1;
    std::vector<Launch> launches_;
    std::vector<Launch> pending_steps_;  // aligned token steps waiting for the in-flight one
    std::map<int, int> slot_of_;
    unsigned long long polls_ = 0;
    double clock_skew_ = 0.0;
    int n_prefill_ = 0, n_decode_ = 0, n_mixed_ = 0;
    std::deque<PromptJob> jobs_;  // fuse mode: prompt tasks in flight as chunks
};

EventLog run_split_engine(const SimulationInputs& inputs, Scheduler& scheduler, sw_model* model, sw_kv* kv,
                          const GpuOptions& options, RunOutputs* outputs) {
    if (!model || !kv) throw ConfigError("run_split_engine: null model or KV arena");
    SW_CUDA(cudaSetDevice(model->device));
    GpuExecutor ex(inputs, scheduler, model, kv, options);
    EventLog log = ex.run();
    if (outputs) ex.collect(*outputs);
    return log;
}

int64_t derive_kv_capacity_pages(const sw_model_desc& d, int device, int64_t reserve_bytes) {
    if (d.n_layers < 1 || d.n_kv_heads < 1 || d.head_dim < 1) throw ConfigError("kv capacity: bad model shape");
    if (reserve_bytes < 0) throw ConfigError("kv capacity: reserve_bytes must be >= 0");
    SW_CUDA(cudaSetDevice(device));
    size_t free_b = 0, total_b = 0;
    SW_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // one page = page_tokens tokens of K and V for every layer and kv head, fp16 (kv_t)
    constexpr int64_t kPageTokens = 16;  // sw_kv::page_tokens
    const int64_t page_bytes = static_cast<int64_t>(d.n_layers) * 2 * d.n_kv_heads * kPageTokens * d.head_dim * 2;
    const int64_t budget = static_cast<int64_t>(free_b) - reserve_bytes;
    return budget > 0 ? budget / page_bytes : 0;
}

// The `#pages` / `#tokens` / `#devpages` / `#gpu` trailer of sw_engine_run's text.
static std::string render_outputs(const EventLog&, const RunOutputs& o) {
    std::string s;
    for (const auto& [rid, toks] : o.tokens) {
        s += "#tokens " + std::to_string(rid) + ":";
        for (std::size_t j = 0; j < toks.size(); ++j) s += (j ? "|" : "") + std::to_string(toks[j]);
        s += "\n";
        s += "#devpages " + std::to_string(rid) + ":";
        const auto& row = o.page_rows.at(rid);
        for (std::size_t j = 0; j < row.size(); ++j) s += (j ? "|" : "") + std::to_string(row[j]);
        s += "\n";
    }
    return s + o.diagnostics;
}

}  // namespace sw

using namespace sw;

extern "C" int sw_engine_run(sw_model* m, sw_kv* kv, const char* spec, char** out) {
    return guarded([&] {
        if (!m || !kv || !spec || !out) throw ConfigError("sw_engine_run: null argument");
        RunSpec rs = build_spec(parse_spec(spec));
        GpuOptions opt;
        for (const auto& [k, v] : rs.rest) {
            if (k == "engine.split") opt.split = v == "1" || v == "true";
            else if (k == "engine.coalesce") opt.coalesce = v == "1" || v == "true";
            else if (k == "engine.align") opt.align = v == "1" || v == "true";
            else if (k == "engine.graphs") opt.graphs = v == "1" || v == "true";
            else if (k == "engine.decode_lanes") opt.decode_lanes = std::stoi(v);
            else if (k == "engine.decode_sms") opt.decode_sms = std::stoi(v);
            else if (k == "engine.lean_prefill") opt.lean_prefill = v == "1" || v == "true";
            else if (k == "engine.prefill_yield") opt.prefill_yield = std::stoi(v);
            else if (k == "engine.prefill_priority") opt.prefill_priority = !(v == "0" || v == "false");
            else if (k == "engine.fuse") opt.fuse = v == "1" || v == "true";
            else if (k == "engine.chunk_tokens") opt.chunk_tokens = std::stoi(v);
            else if (k == "engine.peak_flops") opt.peak_flops = std::stod(v);
            else if (k == "engine.peak_bytes") opt.peak_bytes = std::stod(v);
            else throw ConfigError("spec: unknown key '" + k + "'");
        }
        // the log's capacities are the real peaks (so alone_s is a roofline time)
        rs.inputs.gpu.compute_capacity = opt.peak_flops;
        rs.inputs.gpu.mem_bandwidth = opt.peak_bytes;
        if (rs.kv_capacity_override <= 0) rs.inputs.gpu.kv_capacity_blocks = kv->n_pages;
        if (rs.scheduler.policy == PolicyKind::MultiInstance || rs.scheduler.policy == PolicyKind::PipelinedSplitwiser)
            if (rs.inputs.discipline.mode == SharingDiscipline::Mode::Exclusive && model_instances(rs.scheduler) > 1)
                rs.inputs.discipline.mode = SharingDiscipline::Mode::MpsConcurrent;
        PolicyScheduler sched(rs.inputs.requests, rs.scheduler, rs.inputs.cost.kv_handoff_s);
        RunOutputs outs;
        const auto w0 = std::chrono::steady_clock::now();
        const EventLog log = run_split_engine(rs.inputs, sched, m, kv, opt, &outs);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
        std::string text = serialize_event_log(log);
        try {
            const MetricsReport rep = build_report(log);
            text += render_report(rep);
            if (!rs.output_dir.empty()) write_experiment(rs.output_dir, rs.emit_event_log, log, rep);
        } catch (const ContractViolation& e) {
            g_last_error = std::string("ContractViolation: ") + e.what();
            text += std::string("#report_error ") + e.what() + "\n";
        }
        text += render_pages(outs.pages) + render_outputs(log, outs);
        text += "#wall wall_s=" + fmt17(wall) + "\n";
        *out = dup_text(text);
    });
}

extern "C" int sw_kv_capacity_pages(const sw_model_desc* desc, int device, int64_t reserve_bytes, int64_t* out) {
    return guarded([&] {
        if (!desc || !out) throw ConfigError("sw_kv_capacity_pages: null argument");
        *out = derive_kv_capacity_pages(*desc, device, reserve_bytes);
    });
}

// Executor core: the engine side of the engine<->scheduler contract.
//
// Both backends share this class:
//   * VirtualClockExecutor (below) advances a virtual clock under the
//     reference's proportional-slowdown law.  It exists to prove, byte for
//     byte against the compiled reference, that the policies, KV ledger, log
//     and metrics of this framework behave exactly like splitsim's
//     (engine.hpp:57-500).  The time-sliced discipline models OS
//     time-slicing of separate processes and is out of scope.
//   * GpuExecutor (gpu_executor.cpp) runs real prefill/decode forward passes
//     on two CUDA streams and takes every timestamp from CUDA events.
//
// Contract reproduced here:
//   - capacity split evenly across instances, remainder to the first ones
//     (engine.hpp:65-72); footprint = ceil((in+out)/B) (engine.hpp:94);
//   - prompt activation: every request Waiting, reserve footprints (throws if
//     over capacity), alloc(input), log TaskStart then Kv (engine.hpp:335-387);
//   - token-step completion: generated++, finish -> free + unreserve +
//     RequestFinish, else grow to blocks_for(in+generated); one Kv record per
//     change; then on_task_complete (engine.hpp:284-327);
//   - batch interning per instance (engine.hpp:389-395).
// New on top: a PagePool assigns physical page ids to the same ledger.  A
// prompt takes blocks_for(in) pages; token step g (which writes KV entry
// in+g-1) takes its page at *launch* from the reservation, so the page table
// always covers the entry being written while the ledger stays identical to
// the reference's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <string>
#include <deque>
#include <vector>

#include "event_log.hpp"
#include "kv.hpp"
#include "policy.hpp"
#include "tasks.hpp"

namespace sw {

struct SharingDiscipline {
    enum class Mode { Exclusive, MpsConcurrent, TimeSliced };
    Mode mode = Mode::Exclusive;
    double quantum_s = 0.002;
    double switch_cost_s = 0.0005;
};

inline const char* to_string(SharingDiscipline::Mode m) {
    switch (m) {
        case SharingDiscipline::Mode::Exclusive: return "exclusive";
        case SharingDiscipline::Mode::MpsConcurrent: return "mps_concurrent";
        case SharingDiscipline::Mode::TimeSliced: return "time_sliced";
    }
    return "?";
}

inline void validate(const SharingDiscipline& d) {
    if (d.mode != SharingDiscipline::Mode::TimeSliced) return;
    if (!(d.quantum_s > 0)) throw ConfigError("discipline.quantum_s: must be > 0");
    if (!(d.switch_cost_s >= 0)) throw ConfigError("discipline.switch_cost_s: must be >= 0");
}

struct SimulationInputs {
    std::vector<Request> requests;  // sorted by (arrival_s, id)
    GpuSpec gpu;
    CostModel cost;
    int block_tokens = 16;
    SharingDiscipline discipline;
    // New: one KV quota shared by every instance instead of
    // the reference's even per-instance split (engine.hpp:65-72).  Each
    // instance's pool reports the whole capacity and reserved_blocks() the sum
    // over instances, so the unchanged admission rule (admit_fifo) admits
    // against the shared quota; the worst-case reservations keep the sum of the
    // instances' allocations within it.
    bool shared_kv_pool = false;
};

// A timestamp that may only be known later (GPU events): `ev >= 0` names a
// backend event resolved when the run ends.
struct Stamp {
    double t = 0.0;
    int ev = -1;
};

class ExecutorCore : public EngineView {
public:
    struct Active {
        PhaseTask task;
        double remaining = 1.0;  // virtual clock only
        long long seq = 0;
        int id = 0;
        int device_slot = -1;  // GPU backend bookkeeping
    };

    ExecutorCore(const SimulationInputs& in, Scheduler& sched) : in_(in), sched_(sched) {
        validate(in_.gpu);
        validate(in_.cost);
        validate(in_.discipline);
        const int n = sched_.n_instances();
        if (n < 1) throw ConfigError("scheduler: needs at least one instance");
        if (in_.discipline.mode == SharingDiscipline::Mode::Exclusive && n > 1)
            throw ConfigError("discipline.mode: exclusive requires a single-instance scheduler");
        const long long total = in_.gpu.kv_capacity_blocks;
        for (int i = 0; i < n; ++i) {
            const long long cap = in_.shared_kv_pool ? total : total / n + (i < total % n ? 1 : 0);
            if (cap < 1) throw ConfigError("gpu.kv_capacity_blocks: too small for instance count");
            pools_.emplace_back(in_.block_tokens, cap);
            log_.kv_capacity.push_back(cap);
        }
        pages_ = PagePool(total);
        reserved_.assign(static_cast<std::size_t>(n), 0);
        n_prompt_.assign(static_cast<std::size_t>(n), 0);
        n_step_.assign(static_cast<std::size_t>(n), 0);
        kv_logged_.assign(static_cast<std::size_t>(n), 0);
        last_batch_.assign(static_cast<std::size_t>(n), {-1, {}});
        log_.compute_capacity = in_.gpu.compute_capacity;
        log_.mem_bandwidth = in_.gpu.mem_bandwidth;
        log_.block_tokens = in_.block_tokens;
        log_.discipline = to_string(in_.discipline.mode);
        double prev = 0.0;
        for (const Request& r : in_.requests) {
            if (r.input_tokens < 1 || r.output_tokens < 1)
                throw ConfigError("request " + std::to_string(r.id) + ": token counts must be >= 1");
            if (!(r.arrival_s >= 0.0) || !std::isfinite(r.arrival_s))
                throw ConfigError("request " + std::to_string(r.id) + ": bad arrival");
            if (r.arrival_s < prev) throw ContractViolation("engine: requests not sorted by arrival");
            prev = r.arrival_s;
            Entry e;
            e.req = r;
            e.req.state = RequestState::Waiting;
            e.footprint = pools_[0].blocks_for(static_cast<long long>(r.input_tokens) + r.output_tokens);
            if (!index_.emplace(r.id, static_cast<int>(entries_.size())).second)
                throw ConfigError("request " + std::to_string(r.id) + ": duplicate id");
            entries_.push_back(e);
        }
    }

    // ---- EngineView ----
    double now() const override { return clock_; }
    const Request& request(int id) const override { return entry(id).req; }
    RequestState state(int id) const override { return entry(id).req.state; }
    int generated(int id) const override { return entry(id).generated; }
    const KvBlockPool& pool(int inst) const override { return pools_.at(static_cast<std::size_t>(inst)); }
    long long reserved_blocks(int inst) const override {
        if (in_.shared_kv_pool) {
            long long all = pending_reserve_;  // prompts accepted earlier in this pass
            for (long long r : reserved_) all += r;
            return all;
        }
        return reserved_.at(static_cast<std::size_t>(inst));
    }
    long long footprint_blocks(int id) const override { return entry(id).footprint; }
    int active_count(int inst, TaskKind k) const override {
        return (k == TaskKind::Prompt ? n_prompt_ : n_step_).at(static_cast<std::size_t>(inst));
    }

    const PagePool& pages() const { return pages_; }
    const std::vector<Active>& active() const { return active_; }

protected:
    struct Entry {
        Request req;
        int generated = 0;
        long long footprint = 0;
        int prefilled = 0;          // prompt tokens in the KV cache (chunked prefill)
        bool chunk_active = false;  // a prompt task holding this request is in flight
    };

    Entry& entry(int id) {
        const auto it = index_.find(id);
        if (it == index_.end()) throw ContractViolation("engine: unknown request " + std::to_string(id));
        return entries_[static_cast<std::size_t>(it->second)];
    }
    const Entry& entry(int id) const { return const_cast<ExecutorCore*>(this)->entry(id); }

    // Backend hook: price a task (demand + alone duration).
    virtual PhaseTask price(const TaskRequest& tr, const std::vector<Request>& prompt_batch) {
        if (tr.kind == TaskKind::Prompt) return make_prompt_task(prompt_batch, in_.gpu, in_.cost, tr.instance_id);
        return make_token_step_task(tr.batch, pools_[static_cast<std::size_t>(tr.instance_id)], in_.gpu, in_.cost,
                                    tr.instance_id, tr.extra_overhead_s);
    }

    long long next_seq() { return seq_++; }

    void log_arrival(const Entry& e, Stamp at) {
        LogRecord r;
        r.kind = LogKind::Arrival;
        r.request = e.req.id;
        r.instance = sched_.instance_of(e.req.id);
        r.input_tokens = e.req.input_tokens;
        r.output_tokens = e.req.output_tokens;
        append(r, at);
        sched_.on_arrival(e.req.id);
    }

    // Shared KV quota: a lane admits against the quota without seeing what
    // another lane admitted in the same pass (the unchanged reference lanes
    // reserve at activation), so a prompt that no longer fits waits here, in
    // order, until reservations are released; its TaskStart is logged when it
    // activates.  Lanes that hold reservations are decoding and release them
    // without needing a prompt, so the wait always ends.
    bool fits(const TaskRequest& tr) const {
        if (!in_.shared_kv_pool || tr.kind != TaskKind::Prompt) return true;
        long long need = 0;
        for (int rid : tr.batch)
            if (entry(rid).req.state == RequestState::Waiting) need += entry(rid).footprint;
        return reserved_blocks(tr.instance_id) + need <= pools_.at(static_cast<std::size_t>(tr.instance_id)).capacity();
    }
    // The next pass's tasks: deferred prompts that fit now (in order), then the
    // scheduler's new ones, deferring any prompt that does not fit.
    std::vector<TaskRequest> pass_tasks() {
        std::vector<TaskRequest> out;
        while (!deferred_.empty() && fits(deferred_.front())) {
            out.push_back(deferred_.front());
            deferred_.pop_front();
            reserve_pending(out.back());
        }
        for (const TaskRequest& tr : sched_.next_tasks(*this)) {
            if (deferred_.empty() && fits(tr)) {
                out.push_back(tr);
                reserve_pending(tr);
            } else if (tr.kind == TaskKind::Prompt) {
                deferred_.push_back(tr);
            } else {
                out.push_back(tr);
            }
        }
        pending_reserve_ = 0;
        return out;
    }
    std::size_t deferred_count() const { return deferred_.size(); }

    // Validate, reserve, allocate and log one task; returns its index in active_.
    std::size_t activate(const TaskRequest& tr, Stamp at) {
        if (tr.instance_id < 0 || tr.instance_id >= static_cast<int>(pools_.size()))
            throw ContractViolation("scheduler: task for unknown instance");
        const auto inst = static_cast<std::size_t>(tr.instance_id);
        std::vector<Request> prompt_batch;
        std::vector<int> chunk_begin;
        const bool chunked = tr.kind == TaskKind::Prompt && !tr.chunk_end.empty();
        if (tr.kind == TaskKind::Prompt) {
            if (chunked && tr.chunk_end.size() != tr.batch.size())
                throw ContractViolation("scheduler: prompt chunk ends do not match the batch");
            long long need = 0;
            for (std::size_t i = 0; i < tr.batch.size(); ++i) {
                const Entry& e = entry(tr.batch[i]);
                // a chunk continues a request whose earlier chunks completed (Prompting, none in flight)
                const bool cont = chunked && e.req.state == RequestState::Prompting && e.prefilled > 0 && !e.chunk_active;
                if (e.req.state != RequestState::Waiting && !cont)
                    throw ContractViolation("scheduler: prompt for request not waiting");
                Request r = e.req;  // priced by the tokens this task prefills
                if (chunked) {
                    const int end = tr.chunk_end[i];
                    if (end <= e.prefilled || end > e.req.input_tokens)
                        throw ContractViolation("scheduler: prompt chunk out of range");
                    if (end < e.req.input_tokens && end % kChunkAlign != 0)
                        throw ContractViolation("scheduler: a split prompt chunk must end on a multiple of 128 tokens");
                    r.input_tokens = end - e.prefilled;
                    chunk_begin.push_back(e.prefilled);
                }
                prompt_batch.push_back(r);
                if (e.req.state == RequestState::Waiting) need += e.footprint;
            }
            if (reserved_blocks(static_cast<int>(inst)) + need > pools_[inst].capacity())
                throw ContractViolation("scheduler: prompt batch exceeds KV reservation capacity");
            for (int rid : tr.batch) {
                Entry& e = entry(rid);
                e.chunk_active = true;
                if (e.req.state != RequestState::Waiting) continue;
                e.req.state = RequestState::Prompting;
                reserved_[inst] += e.footprint;
                if (pools_[inst].alloc(rid, e.req.input_tokens) != KvBlockPool::AllocResult::Ok)
                    throw ContractViolation("engine: prompt KV allocation denied despite reservation");
                pages_.grow_to(rid, static_cast<int>(pools_[inst].blocks_for(e.req.input_tokens)));
            }
        } else {
            for (int rid : tr.batch) {
                const Entry& e = entry(rid);
                if (e.req.state != RequestState::Generating)
                    throw ContractViolation("scheduler: token step for request not generating");
                // the entry this step writes is in + generated (0-based)
                const long long pos = static_cast<long long>(e.req.input_tokens) + e.generated;
                pages_.grow_to(rid, static_cast<int>(pools_[inst].blocks_for(pos + 1)));
            }
        }
        Active a;
        a.task = price(tr, prompt_batch);
        if (chunked) {
            a.task.chunk_begin = std::move(chunk_begin);
            a.task.chunk_end = tr.chunk_end;
        }
        a.seq = next_seq();
        a.id = task_counter_++;
        LogRecord r;
        r.kind = LogKind::TaskStart;
        r.task_id = a.id;
        r.instance = tr.instance_id;
        r.task_kind = a.task.kind;
        r.batch_id = intern(tr.instance_id, a.task.batch);
        r.compute = a.task.compute_demand;
        r.mem = a.task.mem_demand;
        r.alone_s = a.task.duration_alone_s;
        append(r, at);
        (a.task.kind == TaskKind::Prompt ? n_prompt_ : n_step_)[inst] += 1;
        active_.push_back(std::move(a));
        if (tr.kind == TaskKind::Prompt) log_kv(tr.instance_id, at);
        return active_.size() - 1;
    }

    void complete(std::size_t idx, Stamp at) {
        const Active done = active_[idx];
        active_.erase(active_.begin() + static_cast<std::ptrdiff_t>(idx));
        const auto inst = static_cast<std::size_t>(done.task.instance_id);
        (done.task.kind == TaskKind::Prompt ? n_prompt_ : n_step_)[inst] -= 1;
        LogRecord r;
        r.kind = LogKind::TaskComplete;
        r.task_id = done.id;
        append(r, at);
        if (done.task.kind == TaskKind::Prompt) {
            for (std::size_t i = 0; i < done.task.batch.size(); ++i) {
                Entry& e = entry(done.task.batch[i]);
                if (e.req.state != RequestState::Prompting)
                    throw ContractViolation("engine: prompt completion for request not prompting");
                e.chunk_active = false;
                e.prefilled = done.task.chunk_end.empty() ? e.req.input_tokens : done.task.chunk_end[i];
                if (e.prefilled == e.req.input_tokens) e.req.state = RequestState::Generating;
            }
        } else {
            for (int rid : done.task.batch) {
                Entry& e = entry(rid);
                if (e.req.state != RequestState::Generating)
                    throw ContractViolation("engine: token step for request not generating");
                if (++e.generated > e.req.output_tokens)
                    throw ContractViolation("engine: generated past output budget");
                if (e.generated == e.req.output_tokens) {
                    e.req.state = RequestState::Finished;
                    pools_[inst].free(rid);
                    pages_.release(rid);
                    reserved_[inst] -= e.footprint;
                    LogRecord f;
                    f.kind = LogKind::RequestFinish;
                    f.request = rid;
                    append(f, at);
                } else if (pools_[inst].alloc(rid, static_cast<long long>(e.req.input_tokens) + e.generated) !=
                           KvBlockPool::AllocResult::Ok) {
                    throw ContractViolation("engine: KV growth denied despite reservation");
                }
            }
            log_kv(done.task.instance_id, at);
        }
        sched_.on_task_complete(done.task, *this);
    }

    void check_all_finished() const {
        for (const Entry& e : entries_)
            if (e.req.state != RequestState::Finished)
                throw ContractViolation("engine: quiescent with unfinished request " + std::to_string(e.req.id));
    }

    void append(LogRecord r, Stamp at) {
        r.time_s = at.t;
        log_.records.push_back(r);
        stamps_.push_back(at.ev);
    }

    // Resolve deferred stamps and restore time order (stable, so records that
    // share a timestamp keep their causal order).
    // Device-clock backends: after resolving the deferred stamps, shift every
    // non-arrival record by the smallest delta >= 0 that puts each prompt at or
    // after its requests' (nominal, host-clock) arrivals.  This absorbs skew
    // between the host clock that paces arrivals and the GPU event clock while
    // keeping every device-measured duration and ordering.  Returns the delta.
    template <class Resolve>
    double finalize_times(Resolve&& resolve, bool align_device_clock = false) {
        bool deferred = false;
        for (std::size_t i = 0; i < log_.records.size(); ++i)
            if (stamps_[i] >= 0) {
                log_.records[i].time_s = resolve(stamps_[i]);
                deferred = true;
            }
        if (!deferred) return 0.0;
        double delta = 0.0;
        if (align_device_clock) {
            for (const LogRecord& r : log_.records) {
                if (r.kind != LogKind::TaskStart || r.task_kind != TaskKind::Prompt) continue;
                for (int rid : log_.batches[static_cast<std::size_t>(r.batch_id)])
                    delta = std::max(delta, entry(rid).req.arrival_s - r.time_s);
            }
            if (delta > 0.0)
                for (LogRecord& r : log_.records)
                    if (r.kind != LogKind::Arrival) r.time_s += delta;
        }
        std::vector<std::size_t> order(log_.records.size());
        for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
            return log_.records[a].time_s < log_.records[b].time_s;
        });
        std::vector<LogRecord> sorted;
        sorted.reserve(order.size());
        for (std::size_t i : order) sorted.push_back(log_.records[i]);
        log_.records.swap(sorted);
        rederive_kv_records();
        return delta;
    }

    // Device-clock backends: the kv records of the time-ordered log, derived with the engine's own
    // ledger rules (engine.hpp:284-387: a prompt allocates blocks_for(in) at its start, a token step
    // grows each request to blocks_for(in + g) or frees it at its last token; one record per change,
    // after the task's records).  The host ledger takes the same steps in host order, which can
    // differ from device order: a prompt queued behind an in-flight launch is accepted (allocated)
    // before that launch's completion is polled, but starts on the device after it.  The host
    // pool's end state is checked against the derived one.
    void rederive_kv_records() {
        std::vector<LogRecord> out;
        out.reserve(log_.records.size());
        std::vector<long long> total(pools_.size(), 0), logged(pools_.size(), 0);
        std::map<int, std::pair<TaskKind, int>> task;  // id -> (kind, batch id)
        std::map<int, int> gen;
        std::map<int, bool> alloc;
        int pending = -1;  // instance whose record follows the current task's records
        auto flush = [&]() {
            if (pending < 0) return;
            const auto i = static_cast<std::size_t>(pending);
            if (total[i] != logged[i]) {
                LogRecord k;
                k.kind = LogKind::Kv;
                k.instance = pending;
                k.kv_blocks = total[i];
                k.time_s = out.back().time_s;
                out.push_back(k);
                logged[i] = total[i];
            }
            pending = -1;
        };
        for (const LogRecord& r : log_.records) {
            if (r.kind == LogKind::Kv) continue;
            if (r.kind != LogKind::RequestFinish) flush();
            out.push_back(r);
            if (r.kind == LogKind::TaskStart) {
                task[r.task_id] = {r.task_kind, r.batch_id};
                if (r.task_kind != TaskKind::Prompt) continue;
                for (int rid : log_.batches.at(static_cast<std::size_t>(r.batch_id))) {
                    if (alloc[rid]) continue;  // a later chunk of a chunked prompt
                    alloc[rid] = true;
                    total.at(static_cast<std::size_t>(r.instance)) += pools_[0].blocks_for(entry(rid).req.input_tokens);
                }
                pending = r.instance;
            } else if (r.kind == LogKind::TaskComplete) {
                const auto& [kind, batch] = task.at(r.task_id);
                if (kind != TaskKind::TokenStep) continue;
                int inst = -1;
                for (int rid : log_.batches.at(static_cast<std::size_t>(batch))) {
                    const Entry& e = entry(rid);
                    inst = sched_.instance_of(rid);
                    const long long in = e.req.input_tokens;
                    const int g = ++gen[rid];
                    auto& t = total.at(static_cast<std::size_t>(inst));
                    if (g == e.req.output_tokens)
                        t -= pools_[0].blocks_for(in + g - 1);
                    else
                        t += pools_[0].blocks_for(in + g) - pools_[0].blocks_for(in + g - 1);
                }
                pending = inst;
            }
        }
        flush();
        log_.records.swap(out);
        for (std::size_t i = 0; i < pools_.size(); ++i)
            if (total[i] != pools_[i].total_allocated())
                throw ContractViolation("engine: device-ordered KV ledger disagrees with the host ledger");
    }

    SimulationInputs in_;
    Scheduler& sched_;
    std::vector<Entry> entries_;
    std::map<int, int> index_;
    std::vector<KvBlockPool> pools_;
    PagePool pages_;
    std::vector<long long> reserved_;
    std::deque<TaskRequest> deferred_;  // shared KV quota: prompts waiting for reservations
    long long pending_reserve_ = 0;     // shared KV quota: footprints accepted in the current pass
    void reserve_pending(const TaskRequest& tr) {
        if (!in_.shared_kv_pool || tr.kind != TaskKind::Prompt) return;
        for (int rid : tr.batch)
            if (entry(rid).req.state == RequestState::Waiting) pending_reserve_ += entry(rid).footprint;
    }
    std::vector<int> n_prompt_, n_step_;
    std::vector<Active> active_;
    double clock_ = 0.0;
    long long seq_ = 0;
    int task_counter_ = 0;
    EventLog log_;
    std::vector<int> stamps_;

private:
    int intern(int inst, const std::vector<int>& batch) {
        auto& cache = last_batch_[static_cast<std::size_t>(inst)];
        if (cache.first >= 0 && cache.second == batch) return cache.first;
        log_.batches.push_back(batch);
        cache = {static_cast<int>(log_.batches.size()) - 1, batch};
        return cache.first;
    }

    void log_kv(int inst, Stamp at) {
        const long long total = pools_[static_cast<std::size_t>(inst)].total_allocated();
        if (total == kv_logged_[static_cast<std::size_t>(inst)]) return;
        kv_logged_[static_cast<std::size_t>(inst)] = total;
        LogRecord r;
        r.kind = LogKind::Kv;
        r.instance = inst;
        r.kv_blocks = total;
        append(r, at);
    }

    std::vector<long long> kv_logged_;
    std::vector<std::pair<int, std::vector<int>>> last_batch_;
};

// Virtual-clock backend: tasks progress at 1/sigma of their alone rate,
// sigma = max(1, sum c_rate/C, sum m_rate/M) over active tasks.  Events at one
// timestamp drain in global sequence order (arrivals were sequenced first),
// then exactly one scheduling pass runs (engine.hpp:101-172, 243-256).
class VirtualClockExecutor final : public ExecutorCore {
public:
    VirtualClockExecutor(const SimulationInputs& in, Scheduler& sched) : ExecutorCore(in, sched) {
        if (in_.discipline.mode == SharingDiscipline::Mode::TimeSliced)
            throw ConfigError("discipline.mode: time_sliced is not modelled by this executor");
    }

    EventLog run() {
        const long long n_arrivals = static_cast<long long>(entries_.size());
        seq_ = n_arrivals;  // arrival i carries sequence number i
        std::size_t next_arrival = 0;
        std::uint64_t events = 0;
        for (;;) {
            const double sigma = slowdown();
            double t_next = std::numeric_limits<double>::infinity();
            bool pending = false;
            if (next_arrival < entries_.size()) {
                t_next = entries_[next_arrival].req.arrival_s;
                pending = true;
            }
            for (const Active& a : active_) {
                const double tc = clock_ + a.remaining * a.task.duration_alone_s * sigma;
                if (tc < t_next) t_next = tc;
                pending = true;
            }
            if (!pending) break;
            if (t_next < clock_) t_next = clock_;
            const double dt = t_next - clock_;
            for (Active& a : active_) {
                const double tc = clock_ + a.remaining * a.task.duration_alone_s * sigma;
                if (tc <= t_next) {
                    a.remaining = 0.0;
                } else if (dt > 0.0 && a.task.duration_alone_s > 0.0) {
                    a.remaining -= dt / (a.task.duration_alone_s * sigma);
                    if (a.remaining < 0.0) a.remaining = 0.0;
                }
            }
            clock_ = t_next;
            for (;;) {
                long long best = -1;
                std::size_t done_idx = 0;
                bool is_done = false;
                if (next_arrival < entries_.size() && entries_[next_arrival].req.arrival_s <= t_next)
                    best = static_cast<long long>(next_arrival);
                for (std::size_t i = 0; i < active_.size(); ++i) {
                    if (active_[i].remaining > 0.0) continue;
                    if (best < 0 || active_[i].seq < best) {
                        best = active_[i].seq;
                        done_idx = i;
                        is_done = true;
                    }
                }
                if (best < 0) break;
                if (++events > 10'000'000ULL) throw ContractViolation("engine: livelock guard tripped after 1e7 events");
                if (is_done) {
                    complete(done_idx, {clock_});
                } else {
                    log_arrival(entries_[next_arrival], {clock_});
                    ++next_arrival;
                }
            }
            for (const TaskRequest& tr : pass_tasks()) activate(tr, {clock_});
        }
        if (deferred_count()) throw ContractViolation("engine: deferred prompt never fit the shared KV quota");
        check_all_finished();
        LogRecord end;
        end.kind = LogKind::RunEnd;
        append(end, {clock_});
        return std::move(log_);
    }

private:
    double slowdown() const {
        double c = 0.0, m = 0.0;
        for (const Active& a : active_) {
            if (a.task.duration_alone_s > 0.0) {
                c += a.task.compute_demand / a.task.duration_alone_s;
                m += a.task.mem_demand / a.task.duration_alone_s;
            }
        }
        double s = 1.0;
        if (c / in_.gpu.compute_capacity > s) s = c / in_.gpu.compute_capacity;
        if (m / in_.gpu.mem_bandwidth > s) s = m / in_.gpu.mem_bandwidth;
        return s;
    }
};

// Drop-in for splitsim::run_simulation (engine.hpp:497-500).
inline EventLog run_simulation(const SimulationInputs& in, Scheduler& sched) {
    VirtualClockExecutor ex(in, sched);
    return ex.run();
}

}  // namespace sw

// GPU test of the C++ engine entry (include/splitwise_engine.hpp): a caller's
// own Scheduler drives real prefill/decode on the B200, as the reference's
// tests drive run_simulation (splitsim/engine.hpp:497-500).
//
//   scripted   a restatement of the reference's ScriptedScheduler
//              (tests/test_util.hpp:71-122): per-request prompt, optionally held
//              until another request's prompt finished, then unbatched steps;
//   policy     a PolicyScheduler built by the caller (mixed batching and the
//              pipelined splitwiser), split and serial co-scheduling;
//   contract   schedulers that break the engine contract get the reference's
//              ContractViolation (engine.hpp:337,346,351), bad inputs ConfigError.
// Every log passes the reference's ledger replay and safety checks
// (tests/property_core.hpp:97-168, restated below), and every schedule yields
// the same greedy tokens per request (prefill/decode rows are batch invariant).
//
// Built by csrc/Makefile into paper_2505_03763_b200/split_engine_test and run
// by tests/test_cpp_engine.py (-m gpu).  Exit code 0 = all checks passed.
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/splitwise_engine.hpp"
#include "../../paper_2505_03763_b200/csrc/host/event_log.hpp"
#include "../../paper_2505_03763_b200/csrc/host/report.hpp"
#include "../../paper_2505_03763_b200/csrc/host/run_text.hpp"

using namespace sw;

static int g_failures = 0;
#define CHECK(cond, ...)                                              \
    do {                                                              \
        if (!(cond)) {                                                \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            std::fprintf(stderr, __VA_ARGS__);                        \
            std::fprintf(stderr, "\n");                               \
            ++g_failures;                                             \
        }                                                             \
    } while (0)

// ---- restatement of the reference's ScriptedScheduler (tests/test_util.hpp:71-122)
class ScriptedScheduler final : public Scheduler {
public:
    struct Item {
        int instance = 0;
        int release_after = -1;  // request id whose prompt must finish first
    };
    ScriptedScheduler(int n, std::map<int, Item> items) : n_(n), items_(std::move(items)) {}
    int n_instances() const override { return n_; }
    int instance_of(int rid) const override { return items_.at(rid).instance; }
    void on_arrival(int rid) override { arrived_.push_back(rid); }
    void on_task_complete(const PhaseTask& t, const EngineView&) override {
        if (t.kind == TaskKind::TokenStep)
            for (int rid : t.batch) stepping_.erase(rid);
    }
    std::vector<TaskRequest> next_tasks(const EngineView& v) override {
        std::vector<TaskRequest> out;
        for (int rid : arrived_) {
            const Item& it = items_.at(rid);
            const RequestState st = v.state(rid);
            if (st == RequestState::Waiting && !prompted_.count(rid)) {
                bool ready = true;
                if (it.release_after >= 0) {
                    const RequestState dep = v.state(it.release_after);
                    ready = dep == RequestState::Generating || dep == RequestState::Finished;
                }
                if (ready) {
                    out.push_back({TaskKind::Prompt, {rid}, it.instance, 0.0});
                    prompted_.insert(rid);
                }
            } else if (st == RequestState::Generating && !stepping_.count(rid)) {
                out.push_back({TaskKind::TokenStep, {rid}, it.instance, 0.0});
                stepping_.insert(rid);
            }
        }
        return out;
    }

private:
    int n_;
    std::map<int, Item> items_;
    std::vector<int> arrived_;
    std::set<int> prompted_, stepping_;
};

// A scheduler that asks for whatever `fn` returns on its first pass.
class OneShotScheduler final : public Scheduler {
public:
    explicit OneShotScheduler(std::function<std::vector<TaskRequest>(const EngineView&)> fn) : fn_(std::move(fn)) {}
    int n_instances() const override { return 1; }
    int instance_of(int) const override { return 0; }
    void on_arrival(int) override {}
    void on_task_complete(const PhaseTask&, const EngineView&) override {}
    std::vector<TaskRequest> next_tasks(const EngineView& v) override {
        if (done_) return {};
        done_ = true;
        return fn_(v);
    }

private:
    std::function<std::vector<TaskRequest>(const EngineView&)> fn_;
    bool done_ = false;
};

// ---- the reference's ledger replay (tests/property_core.hpp:97-145)
static void check_kv_conservation(const EventLog& log, const char* what) {
    std::map<int, std::pair<int, int>> req;
    std::map<int, int> gen, inst_of;
    std::map<int, std::pair<TaskKind, int>> task;
    std::map<int, long long> totals;
    const long long B = log.block_tokens;
    auto blocks_for = [&](long long t) { return (t + B - 1) / B; };
    for (const LogRecord& r : log.records) {
        if (r.kind == LogKind::Arrival) {
            req[r.request] = {r.input_tokens, r.output_tokens};
            gen[r.request] = 0;
        } else if (r.kind == LogKind::TaskStart) {
            task[r.task_id] = {r.task_kind, r.batch_id};
            if (r.task_kind == TaskKind::Prompt)
                for (int rid : log.batches.at(static_cast<std::size_t>(r.batch_id))) {
                    totals[r.instance] += blocks_for(req.at(rid).first);
                    inst_of[rid] = r.instance;
                }
        } else if (r.kind == LogKind::TaskComplete) {
            const auto& [kind, bid] = task.at(r.task_id);
            if (kind != TaskKind::TokenStep) continue;
            for (int rid : log.batches.at(static_cast<std::size_t>(bid))) {
                const auto [in, out] = req.at(rid);
                int& g = gen.at(rid);
                ++g;
                if (g == out)
                    totals[inst_of.at(rid)] -= blocks_for(in + g - 1);
                else
                    totals[inst_of.at(rid)] += blocks_for(in + g) - blocks_for(in + g - 1);
            }
        } else if (r.kind == LogKind::Kv) {
            CHECK(r.kv_blocks == totals[r.instance], "%s: kv ledger diverged at t=%g (%lld vs %lld)", what, r.time_s,
                  r.kv_blocks, totals[r.instance]);
            CHECK(r.kv_blocks <= log.kv_capacity.at(static_cast<std::size_t>(r.instance)), "%s: over capacity", what);
        }
    }
    for (const auto& [inst, t] : totals) CHECK(t == 0, "%s: pool %d not drained (%lld)", what, inst, t);
}

// ---- the reference's safety check (tests/property_core.hpp:147-168)
static void check_safety(const EventLog& log, const char* what) {
    std::map<int, double> start, prompt_end, finish;
    std::map<int, std::pair<TaskKind, int>> task;
    struct Span {
        TaskKind kind;
        int batch;
        double start, end;
    };
    std::vector<Span> spans;
    std::map<int, std::size_t> open;
    for (const LogRecord& r : log.records) {
        if (r.kind == LogKind::TaskStart) {
            open[r.task_id] = spans.size();
            spans.push_back({r.task_kind, r.batch_id, r.time_s, -1});
        } else if (r.kind == LogKind::TaskComplete) {
            spans[open.at(r.task_id)].end = r.time_s;
        } else if (r.kind == LogKind::RequestFinish) {
            finish[r.request] = r.time_s;
        }
    }
    for (const Span& s : spans)
        if (s.kind == TaskKind::Prompt)
            for (int rid : log.batches.at(static_cast<std::size_t>(s.batch))) prompt_end[rid] = s.end;
    for (const Span& s : spans) {
        CHECK(s.end >= s.start, "%s: task ends before it starts", what);
        if (s.kind != TaskKind::TokenStep) continue;
        for (int rid : log.batches.at(static_cast<std::size_t>(s.batch))) {
            CHECK(prompt_end.count(rid), "%s: token step before any prompt (request %d)", what, rid);
            if (prompt_end.count(rid))
                CHECK(s.start + 1e-12 >= prompt_end.at(rid), "%s: step of %d starts before its prompt ends", what, rid);
            if (finish.count(rid)) CHECK(s.start <= finish.at(rid) + 1e-12, "%s: step after finish (%d)", what, rid);
        }
    }
}

static SimulationInputs inputs_of(const std::vector<Request>& reqs, long long capacity) {
    SimulationInputs in;
    in.requests = reqs;
    in.gpu.kv_capacity_blocks = capacity;
    in.block_tokens = 16;
    return in;
}

static void check_run(const EventLog& log, const std::vector<Request>& reqs, const RunOutputs& o,
                      std::map<int, std::vector<int32_t>>& tokens_ref, const char* what) {
    const MetricsReport rep = build_report(log);
    long long want = 0;
    for (const Request& r : reqs) want += r.output_tokens;
    CHECK(rep.total_output_tokens == want, "%s: %lld tokens, want %lld", what, rep.total_output_tokens, want);
    check_kv_conservation(log, what);
    check_safety(log, what);
    // replay through the CSV round trip gives the same report
    const MetricsReport again = build_report(parse_event_log(serialize_event_log(log)));
    CHECK(render_report(again) == render_report(rep), "%s: CSV replay changed the report", what);
    for (const Request& r : reqs) {
        const auto& t = o.tokens.at(r.id);
        CHECK(static_cast<int>(t.size()) == r.output_tokens, "%s: request %d has %zu tokens", what, r.id, t.size());
        for (int32_t x : t) CHECK(x >= 0 && x < 4096, "%s: token %d out of vocab", what, x);
        if (!tokens_ref.count(r.id))
            tokens_ref[r.id] = t;
        else
            CHECK(tokens_ref[r.id] == t, "%s: request %d tokens differ from the first schedule", what, r.id);
        CHECK(o.page_rows.at(r.id).size() == static_cast<std::size_t>((r.input_tokens + r.output_tokens + 15) / 16),
              "%s: request %d device page row has %zu pages", what, r.id, o.page_rows.at(r.id).size());
    }
    std::printf("ok %-40s makespan %.4f s, %lld tokens\n", what, rep.makespan_s, rep.total_output_tokens);
}

template <class E, class F>
static void expect_throw(F&& f, const char* needle, const char* what) {
    try {
        f();
        CHECK(false, "%s: no exception", what);
    } catch (const E& e) {
        CHECK(std::string(e.what()).find(needle) != std::string::npos, "%s: wrong message '%s'", what, e.what());
        std::printf("ok %-40s threw: %s\n", what, e.what());
    } catch (const std::exception& e) {
        CHECK(false, "%s: wrong exception type: %s", what, e.what());
    }
}

int main() {
    // configs[0]'s tiny decoder (paper_2505_03763_b200/shapes.py TINY)
    sw_model_desc d{};
    d.n_layers = 2;
    d.d_model = 256;
    d.n_heads = 4;
    d.n_kv_heads = 2;
    d.head_dim = 64;
    d.ffn_dim = 768;
    d.vocab = 4096;
    d.tied_embeddings = 0;
    d.rope_theta = 500000.f;
    d.norm_eps = 1e-5f;
    d.seed = 1;
    d.max_prefill_tokens = 1024;
    d.max_decode_batch = 16;
    sw_model* m = nullptr;
    sw_kv* kv = nullptr;
    if (sw_model_create(&d, 0, &m) != SW_OK || sw_kv_arena_create(m, 256, 16, 16, 40, &kv) != SW_OK) {
        std::fprintf(stderr, "setup failed: %s\n", sw_last_error());
        return 2;
    }
    int64_t cap = 0;
    CHECK(sw_kv_capacity_pages(&d, 0, 1 << 30, &cap) == SW_OK && cap > 1000, "kv capacity %lld pages", (long long)cap);
    std::printf("ok %-40s %lld pages of %d KiB\n", "derive_kv_capacity_pages", (long long)cap,
                2 * d.n_layers * d.n_kv_heads * 16 * d.head_dim * 2 / 1024);

    std::vector<Request> reqs;
    const int ins[] = {40, 17, 64, 33, 96, 5};
    const int outs[] = {6, 9, 4, 7, 12, 3};
    for (int i = 0; i < 6; ++i) reqs.push_back({i, 0.0, ins[i], outs[i], RequestState::Waiting});
    std::map<int, std::vector<int32_t>> tokens;

    for (bool split : {true, false}) {
        // scripted: requests 1 and 3 wait for 0's and 2's prompts; two instances need the
        // concurrent discipline (the reference's MpsConcurrent; here real streams)
        std::map<int, ScriptedScheduler::Item> items;
        for (int i = 0; i < 6; ++i) items[i] = {i % 2, i % 2 == 1 ? i - 1 : -1};
        ScriptedScheduler sched(2, items);
        SimulationInputs in = inputs_of(reqs, 120);
        in.discipline.mode = SharingDiscipline::Mode::MpsConcurrent;
        GpuOptions opt;
        opt.split = split;
        RunOutputs o;
        const EventLog log = run_split_engine(in, sched, m, kv, opt, &o);
        check_run(log, reqs, o, tokens, split ? "scripted, 2 instances, split" : "scripted, 2 instances, serial");
    }
    for (const char* pol : {"mixed", "pipelined", "sequential", "chunked"}) {
        for (bool split : {true, false}) {
            SchedulerConfig cfg;
            int instances = 1;
            if (std::string(pol) == "mixed") {
                cfg.policy = PolicyKind::MixedBatching;
                cfg.max_batch = 4;
            } else if (std::string(pol) == "pipelined") {
                cfg.policy = PolicyKind::PipelinedSplitwiser;
                cfg.splitwiser_processes = 2;
                cfg.max_batch = 2;
                instances = 2;
            } else if (std::string(pol) == "chunked") {  // 128-token prompt chunks
                cfg.policy = PolicyKind::ChunkedPrefill;
                cfg.chunk_tokens = 128;
                cfg.max_batch = 4;
            } else {
                cfg.policy = PolicyKind::Sequential;
                cfg.max_batch = 3;
            }
            PolicyScheduler sched(reqs, cfg, 0.0);
            SimulationInputs in = inputs_of(reqs, 120);
            if (instances > 1) in.discipline.mode = SharingDiscipline::Mode::MpsConcurrent;
            GpuOptions opt;
            opt.split = split;
            RunOutputs o;
            const EventLog log = run_split_engine(in, sched, m, kv, opt, &o);
            const std::string what = std::string("PolicyScheduler ") + pol + (split ? ", split" : ", serial");
            check_run(log, reqs, o, tokens, what.c_str());
        }
    }

    // contract violations (engine.hpp:337,346,351) and configuration errors
    const SimulationInputs in = inputs_of(reqs, 120);
    expect_throw<ContractViolation>([&] {
        OneShotScheduler s([](const EngineView&) { return std::vector<TaskRequest>{{TaskKind::TokenStep, {0}, 0, 0.0}}; });
        run_split_engine(in, s, m, kv);
    }, "token step for request not generating", "step for a waiting request");
    expect_throw<ContractViolation>([&] {
        OneShotScheduler s([](const EngineView&) {
            return std::vector<TaskRequest>{{TaskKind::Prompt, {0, 1, 2, 3, 4, 5}, 0, 0.0}};
        });
        run_split_engine(inputs_of(reqs, 20), s, m, kv);
    }, "exceeds KV reservation capacity", "prompt batch over the KV reservation");
    expect_throw<ContractViolation>([&] {
        OneShotScheduler s([](const EngineView&) { return std::vector<TaskRequest>{{TaskKind::Prompt, {0}, 3, 0.0}}; });
        run_split_engine(in, s, m, kv);
    }, "unknown instance", "task for an unknown instance");
    expect_throw<ContractViolation>([&] {
        OneShotScheduler s([](const EngineView&) { return std::vector<TaskRequest>{{TaskKind::Prompt, {0}, 0, 0.0}}; });
        run_split_engine(in, s, m, kv);
    }, "quiescent with unfinished request", "scheduler that stalls");
    expect_throw<ConfigError>([&] {
        std::vector<Request> bad = reqs;
        bad[2].output_tokens = 0;
        OneShotScheduler s([](const EngineView&) { return std::vector<TaskRequest>{}; });
        run_split_engine(inputs_of(bad, 120), s, m, kv);
    }, "token counts must be >= 1", "request with no output");
    expect_throw<ConfigError>([&] {
        std::vector<Request> big = reqs;
        big[0].input_tokens = 300;  // 300 + 6 tokens > 16 pages of 16
        OneShotScheduler s([](const EngineView&) { return std::vector<TaskRequest>{}; });
        run_split_engine(inputs_of(big, 120), s, m, kv);
    }, "page-table row", "context longer than the arena rows");

    sw_kv_arena_destroy(kv);
    sw_model_destroy(m);
    if (g_failures) {
        std::fprintf(stderr, "%d check(s) failed\n", g_failures);
        return 1;
    }
    std::printf("all checks passed\n");
    return 0;
}

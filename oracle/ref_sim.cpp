// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Drives the UNMODIFIED reference simulator (headers under
// /root/reference/proj/include/splitsim, compiled in place by oracle/Makefile
// into oracle/_ref/refsim) from the same `key=value;...` run spec the product's
// sw_sim_run takes, and prints the same text: the reference event-log CSV
// (splitsim/event_log.hpp:113-161), a `#report` line and `#request` rows built
// by the reference's build_report (metrics.hpp:178-433).  p50/p99 TTFT/TBT are
// not reference fields; they are computed here with the reference's own
// nearest_rank (metrics.hpp:79-85) over its per-request records.
//
// Usage: refsim '<spec>'     (exit 2 config error, 4 contract violation)
//
// Built a second time as refwrite (-DREF_EXPERIMENT, needs nlohmann/json for
// splitsim/experiment.hpp): `refwrite --write DIR '<spec>'` also writes the
// reference's experiment files (write_experiment, experiment.hpp:194-212, with
// the event log); `refwrite --replay events.csv` writes replay_report.json as
// the reference CLI's replay does (tools/splitsim.cpp:73-85).
#include <cmath>
#include <fstream>
#include <sstream>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "splitsim/engine.hpp"
#include "splitsim/event_log.hpp"
#include "splitsim/metrics.hpp"
#include "splitsim/schedulers.hpp"
#ifdef REF_EXPERIMENT
#include "splitsim/experiment.hpp"
#endif

using namespace splitsim;

static std::map<std::string, std::string> parse(const std::string& text) {
    std::map<std::string, std::string> m;
    std::string cur;
    auto flush = [&] {
        std::string c;
        for (char ch : cur)
            if (!isspace(static_cast<unsigned char>(ch))) c += ch;
        if (!c.empty()) {
            auto eq = c.find('=');
            if (eq == std::string::npos) throw ConfigError("spec: bad item " + c);
            m[c.substr(0, eq)] = c.substr(eq + 1);
        }
        cur.clear();
    };
    for (char ch : text) {
        if (ch == ';') flush();
        else cur += ch;
    }
    flush();
    return m;
}

static PolicyKind policy_of(const std::string& s) {
    if (s == "sequential") return PolicyKind::Sequential;
    if (s == "pipelined_splitwiser") return PolicyKind::PipelinedSplitwiser;
    if (s == "continuous_batching") return PolicyKind::ContinuousBatching;
    if (s == "mixed_batching") return PolicyKind::MixedBatching;
    if (s == "multi_instance") return PolicyKind::MultiInstance;
    throw ConfigError("unknown policy " + s);
}

static TokenRange range_of(const std::string& v) {
    TokenRange r;
    auto dots = v.find("..");
    if (dots == std::string::npos) r.min = r.max = std::stoi(v);
    else {
        r.min = std::stoi(v.substr(0, dots));
        r.max = std::stoi(v.substr(dots + 2));
    }
    return r;
}

static std::string g(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

int main(int argc, char** argv) {
    if (argc == 4 && std::string(argv[1]) == "--prng") {  // refsim --prng <seed> <count>
        SplitMix64 rng(std::stoull(argv[2]));
        for (int i = 0, n = std::stoi(argv[3]); i < n; ++i) std::printf("%llu\n", (unsigned long long)rng.next_u64());
        return 0;
    }
    std::string write_dir;
#ifdef REF_EXPERIMENT
    if (argc == 3 && std::string(argv[1]) == "--replay") {
        try {
            MetricsReport rep = replay_file(argv[2]);
            std::filesystem::path dir = std::filesystem::path(argv[2]).parent_path();
            if (dir.empty()) dir = ".";
            write_file_atomic(dir / "replay_report.json", report_to_json(rep).dump(2) + "\n");
            return 0;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 3;
        }
    }
    if (argc == 4 && std::string(argv[1]) == "--write") {
        write_dir = argv[2];
        argv[1] = argv[3];
        argc = 2;
    }
#endif
    if (argc != 2) {
        std::fprintf(stderr, "usage: refsim '<spec>'\n");
        return 2;
    }
    try {
        auto m = parse(argv[1]);
        WorkloadSpec w;
        SchedulerConfig sc;
        SimulationInputs in;
        double budget = 22016.0, block_unit = 1.0;
        long long pinned = 0;
        std::string trace_path;
        for (auto& [k, v] : m) {
            if (k == "n") w.n_requests = std::stoi(v);
            else if (k == "input") w.input_tokens = range_of(v);
            else if (k == "output") w.output_tokens = range_of(v);
            else if (k == "seed") w.seed = std::stoull(v);
            else if (k == "arrival") {
                if (v == "zero" || v == "all_at_zero") w.arrival = ArrivalAllAtZero{};
                else if (v.rfind("fixed:", 0) == 0) w.arrival = ArrivalFixedInterval{std::stod(v.substr(6))};
                else if (v.rfind("poisson:", 0) == 0) w.arrival = ArrivalPoissonRate{std::stod(v.substr(8))};
                else throw ConfigError("bad arrival");
            } else if (k == "policy") sc.policy = policy_of(v);
            else if (k == "inner") sc.inner = policy_of(v);
            else if (k == "max_batch") sc.max_batch = std::stoi(v);
            else if (k == "P") sc.splitwiser_processes = std::stoi(v);
            else if (k == "n_instances") sc.n_instances = std::stoi(v);
            else if (k == "mode") {
                if (v == "exclusive") in.discipline.mode = SharingDiscipline::Mode::Exclusive;
                else if (v == "mps_concurrent") in.discipline.mode = SharingDiscipline::Mode::MpsConcurrent;
                else if (v == "time_sliced") in.discipline.mode = SharingDiscipline::Mode::TimeSliced;
                else throw ConfigError("bad mode");
            } else if (k == "kv_capacity_blocks") pinned = std::stoll(v);
            else if (k == "block_tokens") in.block_tokens = std::stoi(v);
            else if (k == "compute_capacity") in.gpu.compute_capacity = std::stod(v);
            else if (k == "mem_bandwidth") in.gpu.mem_bandwidth = std::stod(v);
            else if (k == "weight_mem_units") in.gpu.weight_mem_units = std::stod(v);
            else if (k == "shared_weights") in.gpu.shared_weights = (v == "true" || v == "1");
            else if (k == "mem_budget_units") budget = std::stod(v);
            else if (k == "block_mem_unit") block_unit = std::stod(v);
            else if (k == "cost.a_p") in.cost.prompt_compute_per_token = std::stod(v);
            else if (k == "cost.b_p") in.cost.prompt_mem_per_token = std::stod(v);
            else if (k == "cost.a_t") in.cost.token_compute_per_req = std::stod(v);
            else if (k == "cost.w_t") in.cost.token_mem_weight_fraction = std::stod(v);
            else if (k == "cost.b_t") in.cost.token_mem_per_kv_block = std::stod(v);
            else if (k == "cost.prompt_overhead_s") in.cost.prompt_overhead_s = std::stod(v);
            else if (k == "cost.step_overhead_s") in.cost.step_overhead_s = std::stod(v);
            else if (k == "cost.kv_handoff_s") in.cost.kv_handoff_s = std::stod(v);
            else if (k == "trace") trace_path = v;
            else throw ConfigError("unknown key " + k);
        }
        validate(sc);
        if (!trace_path.empty()) {  // config.hpp assemble: parse_trace (request.hpp:134-183)
            std::ifstream f(trace_path);
            if (!f) throw ConfigError("workload.trace: cannot open '" + trace_path + "'");
            std::stringstream ss;
            ss << f.rdbuf();
            in.requests = parse_trace(ss.str());
        } else {
            in.requests = generate(w);
        }
        // derive_kv_capacity (config.hpp:66-79), restated to avoid the json dependency.
        int n_inst = sc.policy == PolicyKind::PipelinedSplitwiser ? sc.splitwiser_processes
                     : sc.policy == PolicyKind::MultiInstance     ? sc.n_instances
                                                                  : 1;
        long long k = pinned;
        if (k <= 0) {
            k = static_cast<long long>(std::floor((budget - in.gpu.weight_mem_units) / block_unit));
            if (!in.gpu.shared_weights && n_inst > 1)
                k -= static_cast<long long>(std::ceil(in.gpu.weight_mem_units * (n_inst - 1) / block_unit));
        }
        in.gpu.kv_capacity_blocks = k;
        PolicyScheduler sched(in.requests, sc, in.cost.kv_handoff_s);
        EventLog log = run_simulation(in, sched);
        MetricsReport r = build_report(log);
#ifdef REF_EXPERIMENT
        if (!write_dir.empty()) {
            ExperimentConfig cfg;
            cfg.output_dir = write_dir;
            cfg.emit_event_log = true;
            write_experiment(cfg, RunResult{log, r});
        }
#endif
        std::vector<double> ttft, tbt;
        for (auto& q : r.requests) {
            ttft.push_back(q.ttft_s);
            if (q.output_tokens >= 2) tbt.push_back(q.tbt_mean_s);
        }
        std::sort(ttft.begin(), ttft.end());
        std::sort(tbt.begin(), tbt.end());
        const double nan = std::numeric_limits<double>::quiet_NaN();
        std::string s = serialize_event_log(log);
        s += "#report n_requests=" + std::to_string(r.n_requests) +
             ";total_output_tokens=" + std::to_string(r.total_output_tokens) + ";makespan_s=" + g(r.makespan_s) +
             ";tokens_per_s=" + g(r.tokens_per_s) + ";requests_per_s=" + g(r.requests_per_s) +
             ";steady_tokens_per_s=" + g(r.steady_tokens_per_s) + ";mean_e2e_s=" + g(r.mean_e2e_s) +
             ";median_e2e_s=" + g(r.median_e2e_s) + ";p99_e2e_s=" + g(r.p99_e2e_s) + ";mean_ttft_s=" + g(r.mean_ttft_s) +
             ";mean_tbt_s=" + g(r.mean_tbt_s) + ";p50_ttft_s=" + g(ttft.empty() ? 0.0 : nearest_rank(ttft, 0.5)) +
             ";p99_ttft_s=" + g(ttft.empty() ? 0.0 : nearest_rank(ttft, 0.99)) +
             ";p50_tbt_s=" + g(tbt.empty() ? nan : nearest_rank(tbt, 0.5)) +
             ";p99_tbt_s=" + g(tbt.empty() ? nan : nearest_rank(tbt, 0.99)) +
             ";mean_batch_elapsed_s=" + g(r.mean_batch_elapsed_s) + ";prompt_elapsed_s=" + g(r.prompt_phase.elapsed_s) +
             ";prompt_mean_kv_pct=" + g(r.prompt_phase.mean_kv_pct) +
             ";prompt_mean_compute_pct=" + g(r.prompt_phase.mean_compute_pct) +
             ";prompt_mean_mem_pct=" + g(r.prompt_phase.mean_mem_pct) + ";token_elapsed_s=" + g(r.token_phase.elapsed_s) +
             ";token_mean_kv_pct=" + g(r.token_phase.mean_kv_pct) +
             ";token_mean_compute_pct=" + g(r.token_phase.mean_compute_pct) +
             ";token_mean_mem_pct=" + g(r.token_phase.mean_mem_pct) + "\n";
        for (auto& q : r.requests)
            s += "#request id=" + std::to_string(q.id) + ";arrival_s=" + g(q.arrival_s) + ";ttft_s=" + g(q.ttft_s) +
                 ";e2e_s=" + g(q.e2e_s) + ";tbt_mean_s=" + g(q.tbt_mean_s) + "\n";
        std::fwrite(s.data(), 1, s.size(), stdout);
        return 0;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "ConfigError: %s\n", e.what());
        return 2;
    } catch (const ParseError& e) {  // exit 2 like the reference CLI (tools/splitsim.cpp:124-139)
        std::fprintf(stderr, "ParseError: %s\n", e.what());
        return 2;
    } catch (const ContractViolation& e) {
        std::fprintf(stderr, "ContractViolation: %s\n", e.what());
        return 4;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
}

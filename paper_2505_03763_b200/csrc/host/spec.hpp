// Run specification: a flat `key=value` list (separated by ';', ',' is not a
// separator, whitespace ignored) that names a workload, a policy and the KV /
// cost geometry.  It is the one config surface of the C-ABI (sw_sim_run,
// sw_engine_run) and deliberately mirrors the reference's JSON config keys
// (config.hpp:139-254, README.md "Configuration reference") so a splitsim
// config maps 1:1:
//   n, input (=a or a..b), output, arrival (zero | fixed:<s> | poisson:<rate>),
//   seed, policy, max_batch, P, n_instances, inner, mode, kv_capacity_blocks,
//   block_tokens, compute_capacity, mem_bandwidth, weight_mem_units,
//   shared_weights, mem_budget_units, block_mem_unit, cost.* (a_p ... kv_handoff_s).
// New keys: trace=<csv> (the reference's workload.trace), kv.shared (one KV quota for all instances, executor.hpp), output_dir /
// emit_event_log (experiment files, experiment_files.hpp), engine.* (GPU executor).
// Unknown keys are a ConfigError naming the key (config.hpp:83-91 behaviour).
#pragma once

#include <cmath>
#include <fstream>
#include <sstream>
#include <map>
#include <string>

#include "executor.hpp"
#include "policy.hpp"
#include "workload.hpp"

namespace sw {

using SpecMap = std::map<std::string, std::string>;

inline SpecMap parse_spec(const std::string& text) {
    SpecMap m;
    std::size_t pos = 0;
    while (pos <= text.size()) {
        const std::size_t end = text.find(';', pos);
        std::string item = text.substr(pos, end == std::string::npos ? std::string::npos : end - pos);
        std::string clean;
        for (char c : item)
            if (c != ' ' && c != '\t' && c != '\n' && c != '\r') clean += c;
        if (!clean.empty()) {
            const auto eq = clean.find('=');
            if (eq == std::string::npos || eq == 0) throw ConfigError("spec: expected key=value, got '" + clean + "'");
            m[clean.substr(0, eq)] = clean.substr(eq + 1);
        }
        if (end == std::string::npos) break;
        pos = end + 1;
    }
    return m;
}

inline PolicyKind parse_policy(const std::string& s, const std::string& where) {
    static const std::pair<const char*, PolicyKind> kNames[] = {
        {"sequential", PolicyKind::Sequential},
        {"pipelined_splitwiser", PolicyKind::PipelinedSplitwiser},
        {"continuous_batching", PolicyKind::ContinuousBatching},
        {"mixed_batching", PolicyKind::MixedBatching},
        {"multi_instance", PolicyKind::MultiInstance},
        {"chunked_prefill", PolicyKind::ChunkedPrefill}};
    for (const auto& [n, k] : kNames)
        if (s == n) return k;
    throw ConfigError(where + ": unknown policy '" + s + "'");
}

struct RunSpec {
    WorkloadSpec workload;
    SchedulerConfig scheduler;
    SimulationInputs inputs;  // requests filled by materialize()
    double mem_budget_units = 22016.0;
    double block_mem_unit = 1.0;
    long long kv_capacity_override = 0;  // 0 = derive
    int shard_index = 0, shard_count = 1;  // request sharding across replicas (GPUs)
    SpecMap rest;                        // backend-specific keys (engine.*, model.*)
    std::string trace_path;              // workload from a trace CSV instead of the generator (config.hpp assemble)
    std::string output_dir;              // non-empty: write the experiment files there (experiment_files.hpp)
    bool emit_event_log = false;         // ... including events.csv
};

// K = floor((budget - weights)/block_unit); duplicated weights cost
// ceil(extra/block_unit) blocks (config.hpp:66-79).
inline long long derive_kv_capacity(double budget, double weights, double block_unit, bool shared, int n_inst,
                                    long long pinned) {
    if (pinned > 0) return pinned;
    if (!(block_unit > 0)) throw ConfigError("gpu.block_mem_unit: must be > 0");
    long long k = static_cast<long long>(std::floor((budget - weights) / block_unit));
    if (!shared && n_inst > 1) k -= static_cast<long long>(std::ceil(weights * (n_inst - 1) / block_unit));
    if (k < 1) throw ConfigError("gpu.mem_budget_units: no KV capacity left after weight accounting");
    return k;
}

inline RunSpec build_spec(const SpecMap& m) {
    RunSpec s;
    auto num = [&](const std::string& k, const std::string& v) -> double {
        try {
            std::size_t used = 0;
            const double d = std::stod(v, &used);
            if (used != v.size()) throw std::invalid_argument(v);
            return d;
        } catch (...) {
            throw ConfigError(k + ": wrong type");
        }
    };
    auto integer = [&](const std::string& k, const std::string& v) -> long long {
        const double d = num(k, v);
        if (d != std::floor(d)) throw ConfigError(k + ": wrong type");
        return static_cast<long long>(d);
    };
    auto range = [&](const std::string& k, const std::string& v) {
        TokenRange r;
        const auto dots = v.find("..");
        if (dots == std::string::npos) {
            r.min = r.max = static_cast<int>(integer(k, v));
        } else {
            r.min = static_cast<int>(integer(k, v.substr(0, dots)));
            r.max = static_cast<int>(integer(k, v.substr(dots + 2)));
        }
        return r;
    };
    auto boolean = [&](const std::string& k, const std::string& v) {
        if (v == "true" || v == "1") return true;
        if (v == "false" || v == "0") return false;
        throw ConfigError(k + ": wrong type");
    };
    bool have_ws = false;
    for (const auto& [k, v] : m) {
        if (k == "n") s.workload.n_requests = static_cast<int>(integer(k, v));
        else if (k == "input") s.workload.input_tokens = range(k, v);
        else if (k == "output") s.workload.output_tokens = range(k, v);
        else if (k == "seed") s.workload.seed = static_cast<std::uint64_t>(std::stoull(v));
        else if (k == "arrival") {
            if (v == "zero" || v == "all_at_zero") s.workload.arrival = ArrivalAllAtZero{};
            else if (v.rfind("fixed:", 0) == 0) s.workload.arrival = ArrivalFixedInterval{num(k, v.substr(6))};
            else if (v.rfind("poisson:", 0) == 0) s.workload.arrival = ArrivalPoissonRate{num(k, v.substr(8))};
            else throw ConfigError("workload.arrival: unknown arrival '" + v + "'");
        } else if (k == "policy") s.scheduler.policy = parse_policy(v, "scheduler.policy");
        else if (k == "inner") s.scheduler.inner = parse_policy(v, "scheduler.inner");
        else if (k == "max_batch") s.scheduler.max_batch = static_cast<int>(integer(k, v));
        else if (k == "P") s.scheduler.splitwiser_processes = static_cast<int>(integer(k, v));
        else if (k == "n_instances") s.scheduler.n_instances = static_cast<int>(integer(k, v));
        else if (k == "chunk_tokens") s.scheduler.chunk_tokens = static_cast<int>(integer(k, v));
        else if (k == "tbt_target_ms") s.scheduler.tbt_target_s = num(k, v) * 1e-3;
        else if (k == "chunk_min") s.scheduler.chunk_min = static_cast<int>(integer(k, v));
        else if (k == "chunk_max") s.scheduler.chunk_max = static_cast<int>(integer(k, v));
        else if (k == "mode") {
            if (v == "exclusive") s.inputs.discipline.mode = SharingDiscipline::Mode::Exclusive;
            else if (v == "mps_concurrent") s.inputs.discipline.mode = SharingDiscipline::Mode::MpsConcurrent;
            else if (v == "time_sliced") s.inputs.discipline.mode = SharingDiscipline::Mode::TimeSliced;
            else throw ConfigError("discipline.mode: unknown mode '" + v + "'");
        } else if (k == "kv_capacity_blocks") s.kv_capacity_override = integer(k, v);
        else if (k == "block_tokens") s.inputs.block_tokens = static_cast<int>(integer(k, v));
        else if (k == "kv.shared") s.inputs.shared_kv_pool = v == "1" || v == "true";
        else if (k == "compute_capacity") s.inputs.gpu.compute_capacity = num(k, v);
        else if (k == "mem_bandwidth") s.inputs.gpu.mem_bandwidth = num(k, v);
        else if (k == "weight_mem_units") s.inputs.gpu.weight_mem_units = num(k, v);
        else if (k == "shared_weights") s.inputs.gpu.shared_weights = boolean(k, v);
        else if (k == "mem_budget_units") s.mem_budget_units = num(k, v);
        else if (k == "block_mem_unit") s.block_mem_unit = num(k, v);
        else if (k == "cost.a_p") s.inputs.cost.prompt_compute_per_token = num(k, v);
        else if (k == "cost.b_p") s.inputs.cost.prompt_mem_per_token = num(k, v);
        else if (k == "cost.a_t") s.inputs.cost.token_compute_per_req = num(k, v);
        else if (k == "cost.w_t") s.inputs.cost.token_mem_weight_fraction = num(k, v);
        else if (k == "cost.b_t") s.inputs.cost.token_mem_per_kv_block = num(k, v);
        else if (k == "cost.prompt_overhead_s") s.inputs.cost.prompt_overhead_s = num(k, v);
        else if (k == "cost.step_overhead_s") s.inputs.cost.step_overhead_s = num(k, v);
        else if (k == "cost.kv_handoff_s") s.inputs.cost.kv_handoff_s = num(k, v);
        else if (k == "shard") {
            const auto slash = v.find('/');
            if (slash == std::string::npos) throw ConfigError("shard: expected <index>/<count>");
            s.shard_index = static_cast<int>(integer(k, v.substr(0, slash)));
            s.shard_count = static_cast<int>(integer(k, v.substr(slash + 1)));
            if (s.shard_count < 1 || s.shard_index < 0 || s.shard_index >= s.shard_count)
                throw ConfigError("shard: index must be in [0, count)");
        } else if (k.rfind("engine.", 0) == 0 || k.rfind("model.", 0) == 0) s.rest[k] = v;
        else if (k == "trace") s.trace_path = v;
        else if (k == "output_dir") s.output_dir = v;  // ExperimentConfig::output_dir (config.hpp:44)
        else if (k == "emit_event_log") s.emit_event_log = v == "1" || v == "true";
        else throw ConfigError("spec: unknown key '" + k + "'");
        have_ws = have_ws || k == "n";
    }
    validate(s.scheduler);
    if (!s.trace_path.empty()) {  // config.hpp assemble: the trace replaces the generated workload
        std::ifstream f(s.trace_path);
        if (!f) throw ConfigError("workload.trace: cannot open '" + s.trace_path + "'");
        std::stringstream ss;
        ss << f.rdbuf();
        s.inputs.requests = parse_trace(ss.str());
    } else {
        s.inputs.requests = generate(s.workload);
    }
    if (s.shard_count > 1) {
        // one replica's share of the trace: round robin by arrival order, the
        // reference's multi_instance_split rule (schedulers.hpp:86-92); ids stay global
        std::vector<Request> mine;
        for (std::size_t i = 0; i < s.inputs.requests.size(); ++i)
            if (static_cast<int>(i % static_cast<std::size_t>(s.shard_count)) == s.shard_index)
                mine.push_back(s.inputs.requests[i]);
        s.inputs.requests.swap(mine);
    }
    s.inputs.gpu.kv_capacity_blocks =
        derive_kv_capacity(s.mem_budget_units, s.inputs.gpu.weight_mem_units, s.block_mem_unit,
                           s.inputs.gpu.shared_weights, model_instances(s.scheduler), s.kv_capacity_override);
    (void)have_ws;
    return s;
}

}  // namespace sw

// Phase tasks: the unit a policy schedules (one prompt batch or one token step
// of a running batch) and how it is priced.
//
// Types and validation mirror splitsim/gpu_model.hpp:15-75,137-189 so a policy
// written against the reference sees identical PhaseTask values.  The pricing
// law (duration_alone = max(compute/C, mem/M) + overhead) is what the virtual
// clock backend runs on; on the GPU backend the same fields carry the task's
// *algorithmic* work instead (FLOPs and HBM bytes of the real forward pass, see
// model_work.hpp) and C/M are the measured tensor and HBM peaks, so
// alone_s is the task's roofline time.
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "base.hpp"
#include "kv.hpp"
#include "workload.hpp"

namespace sw {

struct GpuSpec {
    double compute_capacity = 1.0e6;  // units/s (tensor FLOP/s on the GPU backend)
    double mem_bandwidth = 1.0e5;     // units/s (HBM B/s on the GPU backend)
    long long kv_capacity_blocks = 22000;
    double weight_mem_units = 16.0;
    bool shared_weights = true;
};

struct CostModel {
    double prompt_compute_per_token = 1.0;   // a_p
    double prompt_mem_per_token = 0.01;      // b_p
    double token_compute_per_req = 1.0;      // a_t
    double token_mem_weight_fraction = 1.0;  // w_t
    double token_mem_per_kv_block = 0.01;    // b_t
    double prompt_overhead_s = 0.002;
    double step_overhead_s = 0.001;
    double kv_handoff_s = 0.0;
};

inline void validate(const GpuSpec& g) {
    if (!(g.compute_capacity > 0)) throw ConfigError("gpu.compute_capacity: must be > 0");
    if (!(g.mem_bandwidth > 0)) throw ConfigError("gpu.mem_bandwidth: must be > 0");
    if (g.kv_capacity_blocks < 1) throw ConfigError("gpu.kv_capacity_blocks: must be >= 1");
    if (g.weight_mem_units < 0) throw ConfigError("gpu.weight_mem_units: must be >= 0");
}

inline void validate(const CostModel& c) {
    const std::pair<double, const char*> nonneg[] = {
        {c.prompt_compute_per_token, "prompt_compute_per_token"},
        {c.prompt_mem_per_token, "prompt_mem_per_token"},
        {c.token_compute_per_req, "token_compute_per_req"},
        {c.token_mem_per_kv_block, "token_mem_per_kv_block"},
        {c.prompt_overhead_s, "prompt_overhead_s"},
        {c.step_overhead_s, "step_overhead_s"},
        {c.kv_handoff_s, "kv_handoff_s"},
    };
    for (const auto& [v, name] : nonneg)
        if (!(v >= 0)) throw ConfigError(std::string("cost.") + name + ": must be >= 0");
    if (c.token_mem_weight_fraction < 0 || c.token_mem_weight_fraction > 1)
        throw ConfigError("cost.token_mem_weight_fraction: must be in [0,1]");
}

enum class TaskKind { Prompt, TokenStep };

inline const char* to_string(TaskKind k) { return k == TaskKind::Prompt ? "prompt" : "token_step"; }

struct PhaseTask {
    TaskKind kind = TaskKind::Prompt;
    std::vector<int> batch;
    double compute_demand = 0.0;
    double mem_demand = 0.0;
    double duration_alone_s = 0.0;
    int instance_id = 0;
    // Chunked prefill (new): a prompt task may cover prompt
    // tokens [chunk_begin[i], chunk_end[i]) of batch[i] instead of whole
    // prompts.  Empty = whole prompts (the reference's only form).
    std::vector<int> chunk_begin, chunk_end;
};

inline double roofline_duration(double compute, double mem, const GpuSpec& g, double overhead_s) {
    return std::max(compute / g.compute_capacity, mem / g.mem_bandwidth) + overhead_s;
}

inline void check_batch(const std::vector<int>& batch) {
    if (batch.empty()) throw ContractViolation("phase task: empty batch");
    std::vector<int> ids(batch);
    std::sort(ids.begin(), ids.end());
    if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
        throw ContractViolation("phase task: duplicate request in batch");
}

// Prompt batch priced on the summed input tokens (gpu_model.hpp:154-169).
inline PhaseTask make_prompt_task(const std::vector<Request>& batch, const GpuSpec& g, const CostModel& c,
                                  int instance) {
    PhaseTask t;
    t.kind = TaskKind::Prompt;
    t.instance_id = instance;
    long long tokens = 0;
    t.batch.reserve(batch.size());
    for (const auto& r : batch) {
        t.batch.push_back(r.id);
        tokens += r.input_tokens;
    }
    check_batch(t.batch);
    t.compute_demand = c.prompt_compute_per_token * static_cast<double>(tokens);
    t.mem_demand = c.prompt_mem_per_token * static_cast<double>(tokens);
    t.duration_alone_s = roofline_duration(t.compute_demand, t.mem_demand, g, c.prompt_overhead_s);
    return t;
}

// Token step: weights re-read plus every resident KV block (gpu_model.hpp:173-189).
inline PhaseTask make_token_step_task(const std::vector<int>& batch, const KvBlockPool& pool, const GpuSpec& g,
                                      const CostModel& c, int instance, double extra_overhead_s = 0.0) {
    PhaseTask t;
    t.kind = TaskKind::TokenStep;
    t.instance_id = instance;
    t.batch = batch;
    check_batch(t.batch);
    long long blocks = 0;
    for (int id : t.batch) blocks += pool.allocated(id);
    t.compute_demand = c.token_compute_per_req * static_cast<double>(t.batch.size());
    t.mem_demand = c.token_mem_weight_fraction * g.weight_mem_units +
                   c.token_mem_per_kv_block * static_cast<double>(blocks);
    t.duration_alone_s =
        roofline_duration(t.compute_demand, t.mem_demand, g, c.step_overhead_s + extra_overhead_s);
    return t;
}

}  // namespace sw

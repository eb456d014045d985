// splitwise_engine.hpp -- C++ entry of the B200 split-phase engine: the GPU
// counterpart of the reference's engine entry
//
//     EventLog splitsim::run_simulation(const SimulationInputs&, Scheduler&)
//                                                  (splitsim/engine.hpp:497-500)
//
// A caller builds SimulationInputs and ANY Scheduler (the repo's
// PolicyScheduler, a reference-style ScriptedScheduler, its own policy) exactly
// as for the simulator, and gets back the same EventLog record stream
// (Arrival / TaskStart / TaskComplete / RequestFinish / Kv / RunEnd), now with
// times taken from CUDA events on a B200 running real prefill and decode
// forward passes.  build_report, the CSV writer and the reference tests'
// ledger/safety checks (tests/property_core.hpp:97-168) apply unchanged.
//
// Ownership: the inputs are copied, the Scheduler is held by
// reference for the duration of the call (caller-owned), the model and KV
// arena are created through the C-ABI (include/splitwise.h) and must outlive
// the call.  One host thread per GPU; no scheduler callback runs on a CUDA
// host thread.
//
// Errors keep the reference's taxonomy (splitsim/errors.hpp:9-30): a bad
// configuration throws sw::ConfigError, a scheduler that breaks the engine
// contract (engine.hpp:337,346,351) throws sw::ContractViolation, a CUDA
// launch/runtime failure throws sw::CudaError.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "splitwise.h"
#include "../paper_2505_03763_b200/csrc/host/capi_util.hpp"
#include "../paper_2505_03763_b200/csrc/host/executor.hpp"
#include "../paper_2505_03763_b200/csrc/host/policy.hpp"

namespace sw {

// How the two phases share the GPU (the co-scheduler).
struct GpuOptions {
    bool split = true;        // two streams (prefill || decode) vs one stream (the serial baseline)
    int decode_lanes = 1;     // split mode: concurrent decode streams (instance i -> lane i % lanes)
    int decode_sms = 0;       // split mode: > 0 partitions the SMs with green contexts (decode | prefill)
    bool lean_prefill = false;  // split mode: prompts launched while decode work exists use co-resident GEMM tiles
    int prefill_yield = 0;      // split mode: prompts launched while decode work exists cap GEMM tiles per CTA
    bool prefill_priority = true;   // split mode: prefill stream at the higher stream priority (decode-first
                                    // streams starve prompts under back-to-back steps; engine.prefill_priority=0)
    bool coalesce = true;     // one launch per kind per scheduling pass
    bool align = true;        // a token step requested while another is in flight waits for it and
                              // then runs merged with every other waiting step (one weight pass for all lanes)
    bool graphs = true;       // CUDA graphs for decode steps
    bool fuse = false;        // split mode: fused mixed steps -- a prompt task runs as chunks of whole prompts and
                              // every token step requested meanwhile rides in the next chunk's launch (one weight
                              // stream for both phases)
    int chunk_tokens = 0;     // fuse mode: prompt tokens per chunk (0: as many as the prefill workspace holds)
    double peak_flops = 1.6932e15;  // roofline denominators for the logged alone_s
    double peak_bytes = 6.4469e12;
};

// Optional outputs of a run beside the event log.
struct RunOutputs {
    std::map<int, std::vector<int32_t>> tokens;     // request id -> greedy tokens x_1..x_out
    std::map<int, std::vector<int32_t>> page_rows;  // request id -> device page-table row (pages it held)
    PagePool pages;                                 // host page allocator at the end: final rows + alloc/free journal
    std::string diagnostics;                        // "#gpu key=value;..." launch statistics
};

// The GPU engine entry (drop-in for run_simulation on a B200).
EventLog run_split_engine(const SimulationInputs& inputs, Scheduler& scheduler, sw_model* model, sw_kv* kv,
                          const GpuOptions& options = GpuOptions{}, RunOutputs* outputs = nullptr);

// KV capacity from the device (the reference's
// derive_kv_capacity, config.hpp:66-79, with budget = free HBM): pages of
// page_tokens tokens that fit in cudaMemGetInfo's free bytes minus
// `reserve_bytes` of workspace headroom, for the model's layer/head shape.
int64_t derive_kv_capacity_pages(const sw_model_desc& desc, int device, int64_t reserve_bytes);

}  // namespace sw

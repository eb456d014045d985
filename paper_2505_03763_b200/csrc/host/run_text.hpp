// Text rendering of a finished run: the interchange format of the run-level
// C-ABI.  The event log is the reference CSV (event_log.hpp); the report is a
// flat `#report k=v;...` line of the scalar metrics in %.17g, followed by
// per-request rows (the fields of requests.csv, experiment.hpp:93-108) and the
// physical page journal / page-table rows the oracle replays.
#pragma once

#include <string>

#include "event_log.hpp"
#include "kv.hpp"
#include "report.hpp"

namespace sw {

inline std::string render_report(const MetricsReport& r) {
    auto f = [](double v) { return fmt17(v); };
    std::string s = "#report n_requests=" + std::to_string(r.n_requests) +
                    ";total_output_tokens=" + std::to_string(r.total_output_tokens) + ";makespan_s=" + f(r.makespan_s) +
                    ";tokens_per_s=" + f(r.tokens_per_s) + ";requests_per_s=" + f(r.requests_per_s) +
                    ";steady_tokens_per_s=" + f(r.steady_tokens_per_s) + ";mean_e2e_s=" + f(r.mean_e2e_s) +
                    ";median_e2e_s=" + f(r.median_e2e_s) + ";p99_e2e_s=" + f(r.p99_e2e_s) +
                    ";mean_ttft_s=" + f(r.mean_ttft_s) + ";mean_tbt_s=" + f(r.mean_tbt_s) +
                    ";p50_ttft_s=" + f(r.p50_ttft_s) + ";p99_ttft_s=" + f(r.p99_ttft_s) + ";p50_tbt_s=" + f(r.p50_tbt_s) +
                    ";p99_tbt_s=" + f(r.p99_tbt_s) + ";mean_batch_elapsed_s=" + f(r.mean_batch_elapsed_s) +
                    ";prompt_elapsed_s=" + f(r.prompt_phase.elapsed_s) + ";prompt_mean_kv_pct=" +
                    f(r.prompt_phase.mean_kv_pct) + ";prompt_mean_compute_pct=" + f(r.prompt_phase.mean_compute_pct) +
                    ";prompt_mean_mem_pct=" + f(r.prompt_phase.mean_mem_pct) +
                    ";token_elapsed_s=" + f(r.token_phase.elapsed_s) + ";token_mean_kv_pct=" +
                    f(r.token_phase.mean_kv_pct) + ";token_mean_compute_pct=" + f(r.token_phase.mean_compute_pct) +
                    ";token_mean_mem_pct=" + f(r.token_phase.mean_mem_pct) + "\n";
    for (const auto& q : r.requests)
        s += "#request id=" + std::to_string(q.id) + ";arrival_s=" + f(q.arrival_s) + ";ttft_s=" + f(q.ttft_s) +
             ";e2e_s=" + f(q.e2e_s) + ";tbt_mean_s=" + f(q.tbt_mean_s) + "\n";
    return s;
}

inline std::string render_pages(const PagePool& p) {
    std::string s;
    for (const auto& [rid, row] : p.final_rows()) {
        s += "#pages " + std::to_string(rid) + ":";
        for (std::size_t i = 0; i < row.size(); ++i) s += (i ? "|" : "") + std::to_string(row[i]);
        s += "\n";
    }
    s += "#journal ";
    for (std::size_t i = 0; i < p.journal().size(); ++i)
        s += (i ? "|" : "") + std::to_string(p.journal()[i].request) + ":" + std::to_string(p.journal()[i].pages_after);
    s += "\n";
    return s;
}

}  // namespace sw

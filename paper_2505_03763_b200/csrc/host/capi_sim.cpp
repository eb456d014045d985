// C-ABI: error plumbing and the virtual-clock run entry (sw_sim_run).
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../../include/splitwise.h"
#include "capi_util.hpp"
#include "executor.hpp"
#include "experiment_files.hpp"
#include "report.hpp"
#include "run_text.hpp"
#include "spec.hpp"

namespace sw {
thread_local std::string g_last_error;

char* dup_text(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (p) std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}
}  // namespace sw

extern "C" const char* sw_last_error(void) { return sw::g_last_error.c_str(); }

extern "C" void sw_free(void* p) { std::free(p); }

extern "C" int sw_sim_run(const char* spec, char** out) {
    return sw::guarded([&] {
        if (!spec || !out) throw sw::ConfigError("sw_sim_run: null argument");
        sw::RunSpec rs = sw::build_spec(sw::parse_spec(spec));
        if (!rs.rest.empty()) throw sw::ConfigError("spec: unknown key '" + rs.rest.begin()->first + "'");
        sw::PolicyScheduler sched(rs.inputs.requests, rs.scheduler, rs.inputs.cost.kv_handoff_s);
        sw::VirtualClockExecutor ex(rs.inputs, sched);
        const sw::EventLog log = ex.run();
        const sw::MetricsReport rep = sw::build_report(log);
        if (!rs.output_dir.empty()) sw::write_experiment(rs.output_dir, rs.emit_event_log, log, rep);
        *out = sw::dup_text(sw::serialize_event_log(log) + sw::render_report(rep) + sw::render_pages(ex.pages()));
    });
}

extern "C" int sw_replay(const char* events_path, char** out) {
    return sw::guarded([&] {
        if (!events_path || !out) throw sw::ConfigError("sw_replay: null argument");
        *out = sw::dup_text(sw::render_report(sw::replay_file(events_path)));
    });
}

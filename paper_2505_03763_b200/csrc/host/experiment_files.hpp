// Experiment output files of a run -- the reference's write_experiment
// (splitsim/experiment.hpp:194-212) for both the virtual clock and GPU runs:
//   report.json      report_to_json (experiment.hpp:34-90): keys in insertion
//                    order, 2-space indent, NaN -> null, doubles in shortest
//                    round-trip form
//   requests.csv     requests_csv   (experiment.hpp:99-114)
//   timeseries.csv   timeseries_csv (experiment.hpp:118-160)
//   events.csv       the event log (event_log.hpp:113-161), when emit_event_log
// and replay (experiment.hpp:290-296): parse a written events.csv, rebuild the
// report, write replay_report.json next to it -- the replay-equality check
// (reference tests/test_config.cpp:175-188) applies to GPU runs unchanged.
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "base.hpp"
#include "event_log.hpp"
#include "report.hpp"
#ifdef SW_HAVE_NLOHMANN
#include <json.hpp>
#endif

namespace sw {

// ---------------------------------------------------------------- JSON
// A small JSON value (objects keep insertion order), enough for the report document.
struct JVal {
    enum Kind { Null, Bool, Int, Dbl, Arr, Obj } kind = Null;
    bool b = false;
    long long i = 0;
    double d = 0.0;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;  // insertion order, like the reference's ordered Json
    static JVal num(double v) {
        JVal j;
        j.kind = Dbl;
        j.d = v;
        return j;
    }
    static JVal integer(long long v) {
        JVal j;
        j.kind = Int;
        j.i = v;
        return j;
    }
    static JVal boolean(bool v) {
        JVal j;
        j.kind = Bool;
        j.b = v;
        return j;
    }
    static JVal array() {
        JVal j;
        j.kind = Arr;
        return j;
    }
    static JVal object() {
        JVal j;
        j.kind = Obj;
        return j;
    }
    JVal& operator[](const std::string& k) {
        kind = Obj;
        for (auto& [key, v] : obj)
            if (key == k) return v;
        obj.emplace_back(k, JVal{});
        return obj.back().second;
    }
    void push(JVal v) {
        kind = Arr;
        arr.push_back(std::move(v));
    }
};

// Doubles exactly as the reference's JSON library (nlohmann/json 3.11.3, the
// version its README pins) prints them: its Grisu2 digit generation is not
// always the shortest round trip (e.g. 50.959114812191586 where the shortest
// is 50.95911481219159), so byte-identical report.json needs the same
// routine.  The build defines SW_HAVE_NLOHMANN when the header is present in
// the image; otherwise the shortest digits are laid out the same way (fixed
// notation for decimal exponents in (-4, 15], else d.ddde[+-]XX, integral
// values keep ".0") and differ from the reference only in such last digits.
inline std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
#ifdef SW_HAVE_NLOHMANN
    {
        char nb[64];
        char* end = nlohmann::detail::to_chars(nb, nb + sizeof nb, v);
        return std::string(nb, end);
    }
#endif
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    std::string sci(buf, res.ptr);
    std::string sign;
    if (sci[0] == '-') {
        sign = "-";
        sci = sci.substr(1);
    }
    const auto e = sci.find('e');
    std::string digits = sci.substr(0, e);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = std::stoi(sci.substr(e + 1));
    const int len = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point after the first n digits
    std::string out;
    if (len <= n && n <= 15) {
        out = digits + std::string(static_cast<std::size_t>(n - len), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (len > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
        out += eb;
    }
    return sign + out;
}

inline void json_dump(const JVal& j, std::string& out, int indent, int level) {
    const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
    const std::string pad0(static_cast<std::size_t>(indent * level), ' ');
    switch (j.kind) {
        case JVal::Null: out += "null"; break;
        case JVal::Bool: out += j.b ? "true" : "false"; break;
        case JVal::Int: out += std::to_string(j.i); break;
        case JVal::Dbl: out += json_double(j.d); break;
        case JVal::Arr:
            if (j.arr.empty()) {
                out += "[]";
                break;
            }
            out += "[\n";
            for (std::size_t k = 0; k < j.arr.size(); ++k) {
                out += pad;
                json_dump(j.arr[k], out, indent, level + 1);
                out += k + 1 < j.arr.size() ? ",\n" : "\n";
            }
            out += pad0 + "]";
            break;
        case JVal::Obj: {
            if (j.obj.empty()) {
                out += "{}";
                break;
            }
            out += "{\n";
            std::size_t k = 0;
            for (const auto& [key, v] : j.obj) {
                out += pad + "\"" + key + "\": ";
                json_dump(v, out, indent, level + 1);
                out += ++k < j.obj.size() ? ",\n" : "\n";
            }
            out += pad0 + "}";
            break;
        }
    }
}

// report_to_json (experiment.hpp:34-90): same keys and nesting
inline JVal report_json(const MetricsReport& rep) {
    auto D = JVal::num;
    JVal j = JVal::object();
    j["n_requests"] = JVal::integer(rep.n_requests);
    j["total_output_tokens"] = JVal::integer(rep.total_output_tokens);
    j["makespan_s"] = D(rep.makespan_s);
    JVal thr = JVal::object();
    thr["tokens_per_s"] = D(rep.tokens_per_s);
    thr["requests_per_s"] = D(rep.requests_per_s);
    thr["steady_state_tokens_per_s"] = D(rep.steady_tokens_per_s);
    j["throughput"] = thr;
    JVal lat = JVal::object();
    lat["mean_e2e_s"] = D(rep.mean_e2e_s);
    lat["median_e2e_s"] = D(rep.median_e2e_s);
    lat["p99_e2e_s"] = D(rep.p99_e2e_s);
    lat["mean_ttft_s"] = D(rep.mean_ttft_s);
    lat["mean_tbt_s"] = D(rep.mean_tbt_s);
    j["latency"] = lat;
    auto phase = [&](const PhaseAggregates& p) {
        JVal o = JVal::object();
        o["present"] = JVal::boolean(p.present);
        o["elapsed_s"] = D(p.elapsed_s);
        o["mean_kv_pct"] = D(p.mean_kv_pct);
        o["mean_compute_pct"] = D(p.mean_compute_pct);
        o["mean_mem_pct"] = D(p.mean_mem_pct);
        return o;
    };
    JVal ph = JVal::object();
    ph["prompt"] = phase(rep.prompt_phase);
    ph["token"] = phase(rep.token_phase);
    j["phase"] = ph;
    JVal per_inst = JVal::array();
    for (const auto& inst : rep.batch_elapsed_s) {
        JVal a = JVal::array();
        for (double v : inst) a.push(D(v));
        per_inst.push(a);
    }
    JVal be = JVal::object();
    be["mean_s"] = D(rep.mean_batch_elapsed_s);
    be["per_instance"] = per_inst;
    j["batch_elapsed"] = be;
    JVal reqs = JVal::array();
    for (const auto& r : rep.requests) {
        JVal o = JVal::object();
        o["id"] = JVal::integer(r.id);
        o["instance"] = JVal::integer(r.instance);
        o["arrival_s"] = D(r.arrival_s);
        o["input_tokens"] = JVal::integer(r.input_tokens);
        o["output_tokens"] = JVal::integer(r.output_tokens);
        o["prompt_start_s"] = D(r.prompt_start_s);
        o["first_token_s"] = D(r.first_token_s);
        o["finish_s"] = D(r.finish_s);
        o["ttft_s"] = D(r.ttft_s);
        o["e2e_s"] = D(r.e2e_s);
        o["tbt_mean_s"] = D(r.tbt_mean_s);
        reqs.push(o);
    }
    j["per_request"] = reqs;
    JVal kv = JVal::array();
    for (const auto& series : rep.kv_pct) {
        JVal s = JVal::array();
        for (const auto& p : series) {
            JVal o = JVal::object();
            o["time_s"] = D(p.time_s);
            o["pct"] = D(p.value);
            s.push(o);
        }
        kv.push(s);
    }
    j["kv_series"] = kv;
    JVal util = JVal::array();
    for (const auto& p : rep.util) {
        JVal o = JVal::object();
        o["time_s"] = D(p.time_s);
        o["compute_pct"] = D(p.compute_pct);
        o["mem_pct"] = D(p.mem_pct);
        util.push(o);
    }
    j["util_series"] = util;
    return j;
}

inline std::string report_json_text(const MetricsReport& rep) {
    std::string s;
    json_dump(report_json(rep), s, 2, 0);
    return s + "\n";
}

// requests_csv (experiment.hpp:99-114)
inline std::string requests_csv(const MetricsReport& rep) {
    std::string out = "id,arrival_s,ttft_s,e2e_s,tbt_mean_s\n";
    for (const auto& r : rep.requests)
        out += std::to_string(r.id) + "," + fmt17(r.arrival_s) + "," + fmt17(r.ttft_s) + "," + fmt17(r.e2e_s) + "," +
               fmt17(r.tbt_mean_s) + "\n";
    return out;
}

// timeseries_csv (experiment.hpp:118-160): per-instance rows at the union of
// the instance's KV and utilisation breakpoints, values piecewise constant
inline std::string timeseries_csv(const MetricsReport& rep) {
    struct Row {
        double t;
        int inst;
        double kv, c, m;
    };
    std::vector<Row> rows;
    for (std::size_t i = 0; i < rep.instance_util.size(); ++i) {
        const auto& kv = rep.kv_pct[i];
        const auto& ut = rep.instance_util[i];
        std::vector<double> times;
        for (const auto& p : kv) times.push_back(p.time_s);
        for (const auto& p : ut) times.push_back(p.time_s);
        std::sort(times.begin(), times.end());
        times.erase(std::unique(times.begin(), times.end()), times.end());
        std::size_t ik = 0, iu = 0;
        for (double t : times) {
            while (ik + 1 < kv.size() && kv[ik + 1].time_s <= t) ++ik;
            while (iu + 1 < ut.size() && ut[iu + 1].time_s <= t) ++iu;
            rows.push_back({t, static_cast<int>(i), kv.empty() ? 0.0 : kv[ik].value,
                            ut.empty() ? 0.0 : ut[iu].compute_pct, ut.empty() ? 0.0 : ut[iu].mem_pct});
        }
    }
    std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
        return a.t != b.t ? a.t < b.t : a.inst < b.inst;
    });
    std::string out = "time_s,instance,kv_pct,compute_pct,mem_pct\n";
    for (const auto& r : rows)
        out += fmt17(r.t) + "," + std::to_string(r.inst) + "," + fmt17(r.kv) + "," + fmt17(r.c) + "," + fmt17(r.m) + "\n";
    return out;
}

inline void write_file_atomic(const std::filesystem::path& path, const std::string& content) {
    const std::filesystem::path tmp = path.string() + ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw IoError("cannot write '" + tmp.string() + "'");
        out << content;
        if (!out) throw IoError("write failed for '" + tmp.string() + "'");
    }
    std::error_code ec;
    std::filesystem::rename(tmp, path, ec);
    if (ec) throw IoError("rename to '" + path.string() + "' failed: " + ec.message());
}

// write_experiment (experiment.hpp:194-212)
inline void write_experiment(const std::string& output_dir, bool emit_event_log, const EventLog& log,
                             const MetricsReport& rep) {
    const std::filesystem::path dir(output_dir);
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) throw IoError("cannot create output_dir '" + dir.string() + "': " + ec.message());
    write_file_atomic(dir / "report.json", report_json_text(rep));
    write_file_atomic(dir / "requests.csv", requests_csv(rep));
    write_file_atomic(dir / "timeseries.csv", timeseries_csv(rep));
    if (emit_event_log) write_file_atomic(dir / "events.csv", serialize_event_log(log));
}

// replay (experiment.hpp:290-296 + tools/splitsim.cpp `replay`): report of a
// written event log; replay_report.json is written next to it
inline MetricsReport replay_file(const std::string& events_path) {
    std::ifstream in(events_path);
    if (!in) throw IoError("cannot open event log '" + events_path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const MetricsReport rep = build_report(parse_event_log(ss.str()));
    const std::filesystem::path p(events_path);
    write_file_atomic(p.parent_path() / "replay_report.json", report_json_text(rep));
    return rep;
}

}  // namespace sw

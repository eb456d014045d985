"""Command-line front end in the shape of the reference's `splitsim` CLI
(tools/splitsim.cpp:89-141): `run`, `sweep` and `replay` over the reference's
JSON experiment configs (config.hpp:139-254, README "Configuration reference"),
for the virtual-clock backend (`--backend sim`, sw_sim_run) and the B200 engine
(`--backend gpu`, sw_engine_run on a model of `--model` shape).

  python -m paper_2505_03763_b200.cli run -c configs/hf_splitwiser.json [--set scheduler.P=4] [--emit-events]
  python -m paper_2505_03763_b200.cli run -c cfg.json --backend gpu --model LLAMA_1B --set engine.split=1
  python -m paper_2505_03763_b200.cli sweep -c configs/sweep_batch.json
  python -m paper_2505_03763_b200.cli replay out/run/events.csv [--out dir]
  python -m paper_2505_03763_b200.cli validate -c cfg.json

A config becomes the C-ABI's `key=value;...` run spec (config_to_spec); the
run writes report.json / requests.csv / timeseries.csv (/ events.csv) under
output_dir exactly as the reference's write_experiment does, and prints the
reference's summary line.  Exit codes follow the reference: 2 config error,
3 I/O error, 4 contract violation.  `engine.*` / `kv.shared` keys (this
engine's co-scheduler options) ride along in an
optional top-level "engine" object or through --set.
"""
from __future__ import annotations

import argparse
import copy
import json
import math
import os
import sys
from typing import Dict, List

from . import ConfigError, ContractViolation, IoError, SplitwiseError, replay, sim_run

_COST = {"prompt_compute_per_token": "cost.a_p", "prompt_mem_per_token": "cost.b_p",
         "token_compute_per_req": "cost.a_t", "token_mem_weight_fraction": "cost.w_t",
         "token_mem_per_kv_block": "cost.b_t", "prompt_overhead_s": "cost.prompt_overhead_s",
         "step_overhead_s": "cost.step_overhead_s", "kv_handoff_s": "cost.kv_handoff_s"}
_GPU = ("compute_capacity", "mem_bandwidth", "mem_budget_units", "block_mem_unit", "weight_mem_units",
        "shared_weights", "block_tokens", "kv_capacity_blocks")
_TOP = {"workload", "gpu", "cost", "scheduler", "discipline", "output_dir", "emit_event_log", "seed", "engine"}


def _expect(obj: dict, where: str, keys) -> None:
    for k in obj:
        if k not in keys:
            raise ConfigError(-2, f"{where}: unknown key '{k}'")


def _range(v, where: str) -> str:
    if isinstance(v, bool):
        raise ConfigError(-2, f"{where}: expected an integer or [min, max]")
    if isinstance(v, int):
        return str(v)
    if isinstance(v, list) and len(v) == 2 and all(isinstance(x, int) and not isinstance(x, bool) for x in v):
        return f"{v[0]}..{v[1]}"
    raise ConfigError(-2, f"{where}: expected an integer or [min, max]")


def _num(v) -> str:
    if isinstance(v, bool):
        return "1" if v else "0"
    return repr(v) if isinstance(v, float) else str(v)


def config_to_spec(cfg: dict) -> str:
    """The reference JSON config (config.hpp parse_config) as a run spec."""
    if not isinstance(cfg, dict):
        raise ConfigError(-2, "config: expected a JSON object")
    _expect(cfg, "config", _TOP)
    kv: Dict[str, str] = {}
    seed = cfg.get("seed", 0)
    w = cfg.get("workload")
    if w is None:
        raise ConfigError(-2, "workload: required")
    if "trace" in w:  # the workload from a trace CSV (config.hpp assemble)
        _expect(w, "workload", {"trace"})
        kv["trace"] = w["trace"]
        w = {}
    _expect(w, "workload", {"n_requests", "input_tokens", "output_tokens", "arrival", "seed"})
    if "trace" not in kv:
        kv["n"] = str(w.get("n_requests", 0))
    if "input_tokens" in w:
        kv["input"] = _range(w["input_tokens"], "workload.input_tokens")
    if "output_tokens" in w:
        kv["output"] = _range(w["output_tokens"], "workload.output_tokens")
    kv["seed"] = str(w.get("seed", seed))
    a = w.get("arrival")
    if a is not None:
        if a == "all_at_zero":
            kv["arrival"] = "zero"
        elif isinstance(a, dict) and set(a) == {"fixed_interval_s"}:
            kv["arrival"] = f"fixed:{_num(a['fixed_interval_s'])}"
        elif isinstance(a, dict) and set(a) == {"poisson_rate_per_s"}:
            kv["arrival"] = f"poisson:{_num(a['poisson_rate_per_s'])}"
        else:
            raise ConfigError(-2, "workload.arrival: expected \"all_at_zero\", {fixed_interval_s} or {poisson_rate_per_s}")
    g = cfg.get("gpu", {})
    _expect(g, "gpu", set(_GPU))
    for k in _GPU:
        if k in g:
            kv[k] = _num(g[k])
    c = cfg.get("cost", {})
    _expect(c, "cost", set(_COST))
    for k, sk in _COST.items():
        if k in c:
            kv[sk] = _num(c[k])
    s = cfg.get("scheduler", {})
    # chunk_tokens / tbt_target_ms / chunk_min / chunk_max: policy "chunked_prefill" (new)
    sched_keys = ("policy", "max_batch", "P", "n_instances", "inner", "chunk_tokens", "tbt_target_ms", "chunk_min",
                  "chunk_max")
    _expect(s, "scheduler", set(sched_keys))
    for k in sched_keys:
        if k in s:
            kv[k] = str(s[k])
    d = cfg.get("discipline", {})
    _expect(d, "discipline", {"mode", "quantum_s", "switch_cost_s"})
    if "mode" in d:
        kv["mode"] = d["mode"]
    if d.get("mode") == "time_sliced":
        raise ConfigError(-2, "discipline.mode: time_sliced is out of scope (DESIGN.md section 9)")
    for k, v in (cfg.get("engine") or {}).items():
        kv[k] = _num(v)
    kv["output_dir"] = cfg.get("output_dir", "out")
    if cfg.get("emit_event_log", False):
        kv["emit_event_log"] = "1"
    return ";".join(f"{k}={v}" for k, v in kv.items())


def _parse_value(text: str):
    try:
        return json.loads(text)
    except json.JSONDecodeError:
        return text


def set_path(cfg: dict, path: str, value) -> None:
    """`a.b.c=value` override (config.hpp set_path); engine.* / kv.shared go to the engine object."""
    if path.startswith("engine.") or path == "kv.shared":
        cfg.setdefault("engine", {})[path] = value
        return
    parts = path.split(".")
    cur = cfg
    for p in parts[:-1]:
        cur = cur.setdefault(p, {})
        if not isinstance(cur, dict):
            raise ConfigError(-2, f"--set {path}: '{p}' is not an object")
    cur[parts[-1]] = value


def summary_line(rep: dict) -> str:
    """experiment.hpp summary_line (format_double = %.17g)."""
    f = lambda v: "%.17g" % v  # noqa: E731
    return f"makespan_s={f(rep['makespan_s'])}, tokens_per_s={f(rep['tokens_per_s'])}, mean_ttft_s={f(rep['mean_ttft_s'])}"


class _Runner:
    def __init__(self, backend: str, model: str):
        self.backend = backend
        self.model_name = model
        self.eng = None
        self.sizes = (0, 0, 0, 0)  # (slots, pages per slot, output tokens, decode rows) of the live engine

    def run(self, spec: str, cfg: dict):
        if self.backend == "sim":
            return sim_run(spec)
        from . import runtime, shapes

        # size the engine from this run's actual request list (generated workload or trace file): the
        # virtual-clock backend assembles the same requests in milliseconds; rebuild when a later sweep
        # value needs more slots, longer page-table rows, more output tokens or a wider decode batch
        n, ctx, out = self._extent(spec)
        pages = (ctx + 15) // 16 + 1
        need = (n + 8, pages, out + 1, min(256, max(1, n)))
        if self.eng is not None and any(a > b for a, b in zip(need, self.sizes)):
            self.eng.close()
            self.eng = None
        if self.eng is None:
            desc = getattr(shapes, self.model_name)
            self.sizes = need
            self.eng = runtime.Engine(desc, max_prefill_tokens=32768, max_decode_batch=need[3], n_pages=None,
                                      max_pages=need[0] * pages + 64, n_slots=need[0], max_pages_per_slot=pages,
                                      max_out=need[2])
        return self.eng.run(spec)

    @staticmethod
    def _extent(spec: str):
        """(requests, longest prompt + output, longest output) of the run's request list."""
        sim_spec = ";".join(kv for kv in spec.split(";") if not kv.startswith("engine.")
                            and not kv.startswith("output_dir=") and not kv.startswith("emit_event_log="))
        r = sim_run(sim_spec)
        n, ctx, out = 0, 1, 1
        for line in r.event_log.splitlines():
            if ",arrival," in line:
                kv = dict(x.split("=", 1) for x in line.split(",", 2)[2].split(";"))
                i, o = int(kv["input"]), int(kv["output"])
                n, ctx, out = n + 1, max(ctx, i + o), max(out, o)
        return max(n, 1), ctx, out

    def close(self):
        if self.eng is not None:
            self.eng.close()


def _sanitize(v) -> str:
    s = v if isinstance(v, str) else json.dumps(v)
    return "".join(ch if (ch.isalnum() or ch in "-.") else "_" for ch in s)


def cmd_run(args) -> int:
    with open(args.config) as f:
        cfg = json.load(f)
    for item in args.set or []:
        k, _, v = item.partition("=")
        set_path(cfg, k, _parse_value(v))
    if args.output_dir:
        cfg["output_dir"] = args.output_dir
    if args.emit_events:
        cfg["emit_event_log"] = True
    r = _Runner(args.backend, args.model)
    try:
        res = r.run(config_to_spec(cfg), cfg)
    finally:
        r.close()
    print(summary_line(res.report))
    return 0


def cmd_sweep(args) -> int:
    """experiment.hpp run_sweep: one sub-directory per axis value, sweep.csv at the root; failed values are
    marked and do not stop the others."""
    with open(args.config) as f:
        sw = json.load(f)
    _expect(sw, "sweep", {"base", "base_path", "axis", "values"})
    if "base" in sw:
        base = sw["base"]
    elif "base_path" in sw:
        with open(sw["base_path"]) as f:
            base = json.load(f)
    else:
        raise ConfigError(-2, "sweep.base: required (inline object or base_path)")
    axis, values = sw.get("axis", ""), sw.get("values")
    if not axis:
        raise ConfigError(-2, "sweep.axis: required")
    if not isinstance(values, list) or not values:
        raise ConfigError(-2, "sweep.values: non-empty array required")
    root = base.get("output_dir", "out")
    os.makedirs(root, exist_ok=True)
    for item in getattr(args, "set", None) or []:
        k, _, v = item.partition("=")
        set_path(base, k, _parse_value(v))
    rows: List[str] = ["value,status,makespan_s,tokens_per_s,requests_per_s,steady_tokens_per_s,"
                       "mean_ttft_s,mean_tbt_s,mean_e2e_s,p99_e2e_s,mean_batch_elapsed_s"]
    r = _Runner(args.backend, args.model)
    ok = True
    try:
        for v in values:
            cfg = copy.deepcopy(base)
            set_path(cfg, axis, v)
            cfg["output_dir"] = os.path.join(root, _sanitize(v))
            try:
                rep = r.run(config_to_spec(cfg), cfg).report
                vals = [rep[k] for k in ("makespan_s", "tokens_per_s", "requests_per_s", "steady_tokens_per_s",
                                         "mean_ttft_s", "mean_tbt_s", "mean_e2e_s", "p99_e2e_s",
                                         "mean_batch_elapsed_s")]
                rows.append(_sanitize(v) + ",ok," + ",".join("%.17g" % x if not math.isnan(x) else "nan" for x in vals))
                print(f"{axis}={_sanitize(v)}: {summary_line(rep)}")
            except SplitwiseError as e:
                ok = False
                rows.append(_sanitize(v) + ",failed" + "," * 9)
                print(f"{axis}={_sanitize(v)}: FAILED: {e}")
    finally:
        r.close()
    csv_path = os.path.join(root, "sweep.csv")
    with open(csv_path, "w") as f:
        f.write("\n".join(rows) + "\n")
    print(f"sweep.csv: {csv_path}")
    return 0 if ok else 1  # tools/splitsim.cpp sweep_cmd


def cmd_replay(args) -> int:
    res = replay(args.events)  # writes replay_report.json beside the log
    if args.out:
        import shutil

        os.makedirs(args.out, exist_ok=True)
        src = os.path.join(os.path.dirname(os.path.abspath(args.events)), "replay_report.json")
        shutil.move(src, os.path.join(args.out, "replay_report.json"))
    print(summary_line(res.report))
    return 0


def cmd_validate(args) -> int:
    """tools/splitsim.cpp validate_cmd: schema, policy/discipline and KV-budget checks, trace readable."""
    with open(args.config) as f:
        cfg = json.load(f)
    for item in args.set or []:
        k, _, v = item.partition("=")
        set_path(cfg, k, _parse_value(v))
    spec = config_to_spec(cfg)
    if "trace" in cfg.get("workload", {}):
        with open(cfg["workload"]["trace"]):
            pass
    # the C++ spec builder validates the rest; an empty workload makes it a no-op run
    probe = ";".join(kv for kv in spec.split(";") if not kv.startswith(("output_dir=", "emit_event_log=", "n=",
                                                                          "trace=", "engine.")))
    sim_run(probe + ";n=0")
    print("ok")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="splitwise", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("-c", "--config", required=True)
        p.add_argument("--backend", choices=["sim", "gpu"], default="sim")
        p.add_argument("--model", default="LLAMA_1B", help="model shape for --backend gpu (shapes.py)")
        if name == "run":
            p.add_argument("--set", action="append", help="override a config field: key.path=value")
            p.add_argument("--emit-events", action="store_true")
            p.add_argument("--output-dir", default="")
        if name == "sweep":
            p.add_argument("--set", action="append", help="override a base-config field: key.path=value")
    p = sub.add_parser("validate")
    p.add_argument("-c", "--config", required=True)
    p.add_argument("--set", action="append")
    p = sub.add_parser("replay")
    p.add_argument("events")
    p.add_argument("--out", default="", help="directory for replay_report.json")
    args = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "sweep": cmd_sweep, "replay": cmd_replay, "validate": cmd_validate}[args.cmd](args)
    except (ConfigError, json.JSONDecodeError) as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except (IoError, OSError) as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return 3
    except ContractViolation as e:
        print(f"contract violation: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())

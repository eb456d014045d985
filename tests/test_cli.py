"""The `splitsim`-shaped CLI front end (paper_2505_03763_b200/cli.py).

* the reference's JSON configs map onto run specs whose experiment files are
  byte-identical to the reference writer's (oracle/_ref/refwrite) -- for the
  shipped configs when /root/reference is present, and for inline configs;
* --set overrides, sweep directories + sweep.csv, replay, exit codes 2/3;
* GPU: the same config through the B200 engine (`--backend gpu`).
"""
import json
import os
import subprocess

import pytest

from conftest import ROOT
from paper_2505_03763_b200 import cli

REFWRITE = os.path.join(ROOT, "oracle", "_ref", "refwrite")
REF_CONFIGS = "/root/reference/proj/configs"
FILES = ("report.json", "requests.csv", "timeseries.csv", "events.csv")

INLINE = {
    "workload": {"n_requests": 24, "input_tokens": [64, 400], "output_tokens": [2, 20],
                 "arrival": {"poisson_rate_per_s": 300.0}, "seed": 5},
    "scheduler": {"policy": "mixed_batching", "max_batch": 8},
    "cost": {"kv_handoff_s": 0.0005},
    "output_dir": "unused",
}


def _read(d, f):
    with open(os.path.join(d, f)) as fh:
        return fh.read()


def _check_against_reference(cfg, out):
    if not os.path.exists(REFWRITE):
        pytest.skip("oracle/_ref/refwrite not built")
    spec = ";".join(kv for kv in cli.config_to_spec(cfg).split(";")
                    if not kv.startswith(("output_dir=", "emit_event_log=")))
    ref = str(out) + "_ref"
    assert subprocess.run([REFWRITE, "--write", ref, spec], capture_output=True).returncode == 0
    for f in FILES:
        assert _read(out, f) == _read(ref, f), f


def _run(tmp_path, cfg, *extra):
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / "out"
    code = cli.main(["run", "-c", str(path), "--output-dir", str(out), "--emit-events", *extra])
    return code, out


def test_inline_config_files_match_reference(tmp_path, capsys):
    code, out = _run(tmp_path, INLINE)
    assert code == 0
    assert capsys.readouterr().out.startswith("makespan_s=")
    cfg = dict(INLINE, output_dir=str(out), emit_event_log=True)
    _check_against_reference(cfg, out)


@pytest.mark.parametrize("name", ["hf_sequential", "hf_splitwiser", "vllm_sp", "vllm_mpsx2", "vllm_mpx2"])
def test_shipped_configs_match_reference(tmp_path, name):
    p = os.path.join(REF_CONFIGS, name + ".json")
    if not os.path.exists(p):
        pytest.skip("reference configs not present")
    with open(p) as f:
        cfg = json.load(f)
    if cfg.get("discipline", {}).get("mode") == "time_sliced":
        with pytest.raises(cli.ConfigError):
            cli.config_to_spec(cfg)
        return
    if cfg["workload"].get("n_requests", 0) * cfg["workload"].get("output_tokens", 1) > 40000:
        cfg["workload"]["n_requests"] = 16  # keep the CPU suite fast
    code, out = _run(tmp_path, cfg)
    assert code == 0
    _check_against_reference(dict(cfg, output_dir=str(out), emit_event_log=True), out)


def test_set_override_and_replay(tmp_path, capsys):
    code, out = _run(tmp_path, INLINE, "--set", "scheduler.max_batch=2", "--set", "kv.shared=1")
    assert code == 0
    line = capsys.readouterr().out.strip()
    assert cli.main(["replay", str(out / "events.csv")]) == 0
    assert capsys.readouterr().out.strip() == line
    assert _read(out, "replay_report.json") == _read(out, "report.json")


def test_sweep_dirs_and_csv(tmp_path):
    sweep = {"base": dict(INLINE, output_dir=str(tmp_path / "sw")), "axis": "workload.n_requests",
             "values": [4, 12]}
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps(sweep))
    assert cli.main(["sweep", "-c", str(p)]) == 0
    rows = _read(tmp_path / "sw", "sweep.csv").splitlines()
    assert rows[0].startswith("value,status,makespan_s,tokens_per_s")
    assert [r.split(",")[:2] for r in rows[1:]] == [["4", "ok"], ["12", "ok"]]
    for v in ("4", "12"):
        assert json.loads(_read(tmp_path / "sw" / v, "report.json"))["n_requests"] == int(v)


def test_exit_codes(tmp_path):
    bad = dict(INLINE, bogus=1)
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(bad))
    assert cli.main(["run", "-c", str(p)]) == 2
    assert cli.main(["run", "-c", str(tmp_path / "missing.json")]) == 3
    too_big = dict(INLINE, gpu={"kv_capacity_blocks": 3})
    p.write_text(json.dumps(too_big))
    assert cli.main(["run", "-c", str(p), "--output-dir", str(tmp_path / "o")]) == 4


@pytest.mark.gpu
def test_gpu_backend_run(tmp_path, capsys):
    cfg = {"workload": {"n_requests": 8, "input_tokens": 64, "output_tokens": 8, "arrival": "all_at_zero"},
           "scheduler": {"policy": "pipelined_splitwiser", "P": 2, "max_batch": 4},
           "discipline": {"mode": "mps_concurrent"}, "engine": {"engine.split": 1}}
    code, out = _run(tmp_path, cfg, "--backend", "gpu", "--model", "TINY")
    assert code == 0
    rep = json.loads(_read(out, "report.json"))
    assert rep["total_output_tokens"] == 64
    assert cli.main(["replay", str(out / "events.csv")]) == 0
    assert _read(out, "replay_report.json") == _read(out, "report.json")


@pytest.mark.gpu
def test_gpu_backend_chunked_prefill(tmp_path):
    """chunked_prefill through the JSON front end on the B200 engine: prompts of 130-300 tokens cut
    into 128-token chunks fused with the token steps; the written log replays to its report."""
    cfg = {"workload": {"n_requests": 6, "input_tokens": [130, 300], "output_tokens": [4, 9], "arrival": "all_at_zero"},
           "scheduler": {"policy": "chunked_prefill", "max_batch": 4, "chunk_tokens": 128},
           "engine": {"engine.split": 1, "engine.fuse": 1}}
    code, out = _run(tmp_path, cfg, "--backend", "gpu", "--model", "TINY")
    assert code == 0
    rep = json.loads(_read(out, "report.json"))
    assert rep["n_requests"] == 6
    assert cli.main(["replay", str(out / "events.csv")]) == 0
    assert _read(out, "replay_report.json") == _read(out, "report.json")


def test_trace_workload_config(tmp_path):
    trace = tmp_path / "trace.csv"
    trace.write_text("id,arrival_s,input_tokens,output_tokens\n0,0.0,100,5\n1,0.001,300,9\n2,0.001,50,2\n")
    cfg = {"workload": {"trace": str(trace)}, "scheduler": {"policy": "mixed_batching"}}
    code, out = _run(tmp_path, cfg)
    assert code == 0
    assert json.loads(_read(out, "report.json"))["n_requests"] == 3
    _check_against_reference(dict(cfg, output_dir=str(out), emit_event_log=True), out)


def test_validate(tmp_path, capsys):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(INLINE))
    assert cli.main(["validate", "-c", str(p)]) == 0
    assert capsys.readouterr().out.strip() == "ok"
    p.write_text(json.dumps(dict(INLINE, scheduler={"policy": "nope"})))
    assert cli.main(["validate", "-c", str(p)]) == 2
    p.write_text(json.dumps(dict(INLINE, scheduler={"policy": "multi_instance", "n_instances": 2},
                                 discipline={"mode": "exclusive"})))
    assert cli.main(["validate", "-c", str(p)]) == 2


def test_gpu_runner_sizes_from_the_request_list(tmp_path):
    """The B200 backend sizes its engine from each run's own request list (the
    reference's sweep over workload.n_requests, configs/sweep_batch.json, and
    trace workloads): _extent reads it off the virtual-clock assembly."""
    spec = cli.config_to_spec(dict(INLINE, output_dir=""))
    n, ctx, out = cli._Runner._extent(spec + ";engine.split=1")
    assert n == 24 and 64 + 2 <= ctx <= 400 + 20 and 2 <= out <= 20
    trace = tmp_path / "trace.csv"
    trace.write_text("id,arrival_s,input_tokens,output_tokens\n0,0.0,100,5\n1,0.001,300,9\n2,0.001,50,2\n")
    n, ctx, out = cli._Runner._extent(cli.config_to_spec({"workload": {"trace": str(trace)},
                                                           "scheduler": {"policy": "mixed_batching"}}))
    assert (n, ctx, out) == (3, 309, 9)


@pytest.mark.gpu
def test_gpu_backend_sweep_grows_the_engine(tmp_path):
    """a B200-backend sweep over n_requests (10 -> 160) and a trace
    workload both run (the engine is rebuilt when a value needs more capacity)."""
    base = {"workload": {"n_requests": 10, "input_tokens": [16, 64], "output_tokens": [2, 6], "seed": 3,
                         "arrival": "all_at_zero"},
            "scheduler": {"policy": "continuous_batching", "max_batch": 0},
            "engine": {"engine.split": 1}, "output_dir": str(tmp_path / "sw")}
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps({"base": base, "axis": "workload.n_requests", "values": [10, 40, 160]}))
    assert cli.main(["sweep", "-c", str(p), "--backend", "gpu", "--model", "TINY"]) == 0
    rows = _read(tmp_path / "sw", "sweep.csv").splitlines()
    assert [r.split(",")[:2] for r in rows[1:]] == [["10", "ok"], ["40", "ok"], ["160", "ok"]]
    trace = tmp_path / "trace.csv"
    trace.write_text("id,arrival_s,input_tokens,output_tokens\n0,0.0,100,5\n1,0.001,300,9\n2,0.001,50,2\n")
    cfg = {"workload": {"trace": str(trace)}, "scheduler": {"policy": "mixed_batching"}}
    code, out = _run(tmp_path, cfg, "--backend", "gpu", "--model", "TINY")
    assert code == 0
    assert json.loads(_read(out, "report.json"))["total_output_tokens"] == 16


def test_chunked_prefill_config_and_replay(tmp_path, capsys):
    """The new chunked_prefill policy through the JSON front end, a --set sweep of its
    budget, and replay of the written event log to the same report."""
    cfg = dict(INLINE, scheduler={"policy": "chunked_prefill", "max_batch": 8, "chunk_tokens": 256})
    code, out = _run(tmp_path, cfg, "--set", "scheduler.chunk_tokens=128")
    assert code == 0
    line = capsys.readouterr().out.strip()
    assert cli.main(["replay", str(out / "events.csv")]) == 0
    assert capsys.readouterr().out.strip() == line
    assert _read(out, "replay_report.json") == _read(out, "report.json")
    cfg["scheduler"] = {"policy": "chunked_prefill", "chunk_tokens": 0, "tbt_target_ms": 5.0}
    code, _ = _run(tmp_path, cfg)
    assert code == 0
    cfg["scheduler"] = {"policy": "chunked_prefill", "chunk_tokens": 100}
    code, _ = _run(tmp_path, cfg)
    assert code == 2  # ConfigError

"""Experiment output files and replay.

The product writes the reference's experiment files for any run when the spec
carries `output_dir=...;emit_event_log=1` (host/experiment_files.hpp, the
reference's write_experiment, experiment.hpp:194-212), and sw_replay rebuilds
a report from a written events.csv (experiment.hpp:290-296).  Checked against
the UNMODIFIED reference writer/replay (oracle/_ref/refwrite):
  * report.json, requests.csv, timeseries.csv, events.csv byte-identical for
    the same virtual-clock run;
  * replay equality (reference tests/test_config.cpp:175-188): replay_report.json
    == report.json, for our replay of our log and the reference's replay of it;
  * recorded reference hashes (tests/golden/sched_golden.json "files:*") when
    refwrite is absent;
  * GPU: an engine run's files replay to the same report, by both replays.
"""
import hashlib
import json
import os
import subprocess

import pytest

from conftest import ROOT
from test_sched_parity import random_spec

REFWRITE = os.path.join(ROOT, "oracle", "_ref", "refwrite")
FILES = ("report.json", "requests.csv", "timeseries.csv", "events.csv")
with open(os.path.join(ROOT, "tests", "golden", "sched_golden.json")) as _f:
    GOLD = {k: v for k, v in json.load(_f).items() if k.startswith("files:")}

SPECS = [
    "n=3;input=20;output=3;seed=1;policy=continuous_batching",
    "n=40;input=10..300;output=1..20;seed=5;arrival=poisson:200;policy=mixed_batching",
    "n=30;input=64;output=8;seed=2;policy=pipelined_splitwiser;P=3;max_batch=4;mode=mps_concurrent",
    "n=24;input=100..400;output=4..12;seed=9;policy=multi_instance;n_instances=2;inner=continuous_batching;"
    "mode=mps_concurrent",
] + [random_spec(2000 + s) for s in range(12)]


def _read(d, f):
    with open(os.path.join(d, f)) as fh:
        return fh.read()


def _ref_write(d, spec):
    if not os.path.exists(REFWRITE):
        pytest.skip("oracle/_ref/refwrite not built")
    p = subprocess.run([REFWRITE, "--write", d, spec], capture_output=True, text=True)
    return p.returncode


@pytest.mark.parametrize("i", range(len(SPECS)))
def test_files_byte_identical_to_reference_writer(swlib, tmp_path, i):
    spec = SPECS[i]
    code = _ref_write(str(tmp_path / "ref"), spec)
    if code != 0:
        with pytest.raises(swlib.SplitwiseError):
            swlib.sim_run(spec)
        return
    swlib.sim_run(spec + f";output_dir={tmp_path / 'mine'};emit_event_log=1")
    for f in FILES:
        assert _read(tmp_path / "mine", f) == _read(tmp_path / "ref", f), (spec, f)


@pytest.mark.parametrize("i", range(4))
def test_replay_equality_both_ways(swlib, tmp_path, i):
    spec = SPECS[i]
    swlib.sim_run(spec + f";output_dir={tmp_path};emit_event_log=1")
    report = _read(tmp_path, "report.json")
    swlib.replay(str(tmp_path / "events.csv"))
    assert _read(tmp_path, "replay_report.json") == report
    if os.path.exists(REFWRITE):
        os.remove(tmp_path / "replay_report.json")
        assert subprocess.run([REFWRITE, "--replay", str(tmp_path / "events.csv")]).returncode == 0
        assert _read(tmp_path, "replay_report.json") == report


@pytest.mark.parametrize("name", sorted(GOLD))
def test_files_match_recorded_reference_hashes(swlib, tmp_path, name):
    g = GOLD[name]
    swlib.sim_run(g["spec"] + f";output_dir={tmp_path};emit_event_log=1")
    for f, h in g["sha256"].items():
        assert hashlib.sha256(_read(tmp_path, f).encode()).hexdigest() == h, (name, f)


def test_replay_of_missing_file_is_io_error(swlib, tmp_path):
    with pytest.raises(swlib.IoError):
        swlib.replay(str(tmp_path / "nope.csv"))


@pytest.mark.gpu
def test_gpu_run_files_replay_to_the_same_report(tmp_path):
    from oracle import model as M
    from paper_2505_03763_b200 import runtime

    eng = runtime.Engine(M.TINY, max_prefill_tokens=1024, max_decode_batch=16, n_pages=512, n_slots=16,
                         max_pages_per_slot=8, max_out=40)
    try:
        eng.run("n=8;input=64;output=32;seed=1;kv_capacity_blocks=480;policy=pipelined_splitwiser;P=2;max_batch=4;"
                f"engine.split=1;output_dir={tmp_path};emit_event_log=1")
    finally:
        eng.close()
    import paper_2505_03763_b200 as sw

    report = _read(tmp_path, "report.json")
    assert json.loads(report)["total_output_tokens"] == 8 * 32
    sw.replay(str(tmp_path / "events.csv"))
    assert _read(tmp_path, "replay_report.json") == report
    if os.path.exists(REFWRITE):  # the reference's own replay of a GPU run's log
        os.remove(tmp_path / "replay_report.json")
        assert subprocess.run([REFWRITE, "--replay", str(tmp_path / "events.csv")]).returncode == 0
        assert _read(tmp_path, "replay_report.json") == report


def test_replay_of_recorded_gpu_log_matches_reference_bytes(swlib, tmp_path):
    """A GPU run's events.csv (irregular device timestamps) once exposed a
    last-digit difference: the reference prints doubles with nlohmann's Grisu2,
    which is not always the shortest round trip.  The recorded reference replay
    of that log (oracle/_ref/refwrite --replay) is the fixture."""
    import shutil

    shutil.copy(os.path.join(ROOT, "tests", "golden", "gpu_run_events.csv"), tmp_path / "events.csv")
    swlib.replay(str(tmp_path / "events.csv"))
    assert _read(tmp_path, "replay_report.json") == _read(os.path.join(ROOT, "tests", "golden"),
                                                           "gpu_run_events.reference_replay.json")

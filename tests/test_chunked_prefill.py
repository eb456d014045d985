"""Chunked prefill policy (new: `policy=chunked_prefill`) on
the virtual-clock backend: the same ExecutorCore and lane the GPU engine runs.

The lane (csrc/host/policy.hpp ChunkLane) cuts prompt tasks into chunks of at
most C prompt tokens, splitting a prompt only at multiples of 128 tokens, and
issues each chunk beside the running set's token step (schedulers.hpp:215-261's
mixed lane is the starting point).  Checked here:
  * every request completes with its token count; the KV ledger replays
    (a chunked prompt is allocated once, by its first chunk);
  * safety: no token step of a request starts before its LAST chunk completed;
  * a prompt of L tokens appears in ceil(L / C) or ceil(L / C) + 1 prompt
    tasks (continuations get the budget first, only the first piece is short);
  * the adaptive controller (chunk_tokens=0): a tighter time-between-tokens
    target yields more, smaller chunks;
  * bad configurations raise ConfigError.
"""
import math

import pytest

import paper_2505_03763_b200 as sw
from oracle import pages as P

BASE = "n=24;input=100..900;output=4..12;seed=7;arrival=poisson:400;max_batch=8"


def _spans(r):
    starts, spans, batches, finish = {}, [], {}, {}
    for line in r.event_log.splitlines()[1:]:
        t, kind, detail = line.split(",", 2)
        kv = dict(x.split("=", 1) for x in detail.split(";") if "=" in x)
        if kind == "batch_def":
            batches[int(kv["batch"])] = [int(x) for x in kv["reqs"].split("|") if x]
        elif kind == "task_start":
            starts[int(kv["task"])] = (kv["kind"], int(kv["batch"]), float(t))
        elif kind == "task_complete":
            k, b, t0 = starts[int(kv["task"])]
            spans.append((k, batches[b], t0, float(t)))
        elif kind == "request_finish":
            finish[int(kv["req"])] = float(t)
    return spans, finish


def _arrivals(r):
    req = {}
    for line in r.event_log.splitlines():
        if ",arrival," in line:
            kv = dict(x.split("=", 1) for x in line.split(",", 2)[2].split(";"))
            req[int(kv["req"])] = (int(kv["input"]), int(kv["output"]))
    return req


@pytest.mark.parametrize("chunk", [128, 256, 1000, 4096])
def test_chunked_runs_complete_safely(chunk):
    r = sw.sim_run(f"{BASE};policy=chunked_prefill;chunk_tokens={chunk}")
    req = _arrivals(r)
    assert r.report["n_requests"] == len(req)
    assert r.report["total_output_tokens"] == sum(o for _, o in req.values())
    last = {}
    for t, inst, logged, replayed in P.ledger_replay(r.event_log):
        assert logged == replayed, t
        last[inst] = logged
    assert all(v == 0 for v in last.values())
    spans, finish = _spans(r)
    prompt_end, n_prompt_tasks = {}, {}
    for k, b, t0, t1 in spans:
        if k == "prompt":
            for rid in b:
                prompt_end[rid] = max(prompt_end.get(rid, 0.0), t1)
                n_prompt_tasks[rid] = n_prompt_tasks.get(rid, 0) + 1
    for k, b, t0, t1 in spans:
        if k == "token_step":
            for rid in b:
                assert t0 + 1e-12 >= prompt_end[rid], rid
                assert t0 <= finish[rid] + 1e-12
    for rid, (i, _) in req.items():
        # continuations get the whole budget first; only a prompt's first piece can be short
        assert math.ceil(i / chunk) <= n_prompt_tasks[rid] <= math.ceil(i / chunk) + 1, (rid, i)


def test_adaptive_budget_follows_the_target():
    # virtual clock: the chunk task's duration grows with its tokens, so a tighter TBT target
    # settles on smaller chunks (more prompt tasks for the same prompts)
    n_tasks = []
    for target in (2.0, 50.0):
        r = sw.sim_run(f"{BASE};policy=chunked_prefill;chunk_tokens=0;tbt_target_ms={target}")
        spans, _ = _spans(r)
        n_tasks.append(sum(1 for k, *_ in spans if k == "prompt"))
        assert r.report["total_output_tokens"] == sum(o for _, o in _arrivals(r).values())
    assert n_tasks[0] > n_tasks[1], n_tasks


def test_chunked_inside_multi_instance():
    r = sw.sim_run(f"{BASE};policy=multi_instance;n_instances=2;inner=chunked_prefill;chunk_tokens=256;mode=mps_concurrent")
    assert r.report["total_output_tokens"] == sum(o for _, o in _arrivals(r).values())


@pytest.mark.parametrize("bad", ["chunk_tokens=100", "chunk_tokens=-1", "tbt_target_ms=0",
                                 "chunk_tokens=0;chunk_min=64", "chunk_tokens=0;chunk_min=512;chunk_max=256"])
def test_bad_chunk_config(bad):
    with pytest.raises(sw.ConfigError):
        sw.sim_run(f"{BASE};policy=chunked_prefill;{bad}")

"""End-to-end GPU runs through sw_engine_run (the run-level C-ABI).

Config 1 of BASELINE.json (tiny decoder, 8 prompts x 64 tokens, 32 greedy
steps) under serial and split-phase policies:
  * every policy/mode yields the same tokens (batch-invariant kernels), and
    each token agrees with the fp32 oracle (teacher forced) wherever the
    oracle's top-2 margin exceeds the 1e-2 tolerance;
  * the device page table equals the host allocator's rows and an
    independent replay of the alloc/free journal (bit exact);
  * the event log obeys the reference contract (KV ledger replay, token
    counts, one TTFT/TBT per request).
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import model as M
from oracle import pages as P

pytestmark = pytest.mark.gpu

RUNS = {
    "sequential_serial": "policy=sequential;max_batch=8;engine.split=0",
    "cb_serial": "policy=continuous_batching;engine.split=0",
    "pipelined_P2_split": "policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1",
    "pipelined_P4_split_nocoalesce": "policy=pipelined_splitwiser;P=4;max_batch=2;engine.split=1;engine.coalesce=0",
    "mixed_split_arrivals": "policy=mixed_batching;arrival=fixed:0.003;engine.split=1",
    "multi_instance_split": "policy=multi_instance;n_instances=2;inner=mixed_batching;engine.split=1",
    # co-scheduler on green-context SM partitions (decode 48 SMs | prefill the rest)
    "pipelined_P2_green48": "policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1;engine.decode_lanes=2;"
                            "engine.decode_sms=48",
    "mixed_green64_arrivals": "policy=mixed_batching;arrival=fixed:0.003;engine.split=1;engine.decode_sms=64",
    # prefill GEMMs capped at one tile per CTA while decode work exists (tile-granular interleaving)
    "pipelined_P2_yield1": "policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1;engine.prefill_yield=1",
    "pipelined_P2_prefill_priority": "policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1;"
                                     "engine.prefill_priority=1",
    # prompts launched while decode work exists on lean CTA-pair GEMMs (co-resident with decode CTAs)
    "pipelined_P2_lean": "policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1;engine.lean_prefill=1",
    # fused mixed steps: prompts in chunks of <= 96 tokens, token steps riding in the chunks' launches
    "mixed_fused_chunks": "policy=mixed_batching;arrival=fixed:0.0005;engine.split=1;engine.fuse=1;engine.chunk_tokens=96",
}
FUSED = {"mixed_fused_chunks"}  # decode rows through the prefill GEMMs: oracle parity, not bit identity


@pytest.fixture(scope="module")
def eng():
    from paper_2505_03763_b200 import runtime

    e = runtime.Engine(M.TINY, max_prefill_tokens=1024, max_decode_batch=16, n_pages=512, n_slots=16,
                       max_pages_per_slot=8, max_out=40)
    yield e
    e.close()


@pytest.fixture(scope="module")
def results(eng):
    out = {}
    for name, extra in RUNS.items():
        out[name] = eng.run(f"n=8;input=64;output=32;seed=1;kv_capacity_blocks=480;{extra}")
    return out


def test_all_runs_complete(results):
    for name, r in results.items():
        assert r.report["n_requests"] == 8, name
        assert r.report["total_output_tokens"] == 8 * 32, name
        assert len(r.tokens) == 8 and all(len(t) == 32 for t in r.tokens.values()), name


def test_tokens_identical_across_policies_and_modes(results):
    base = results["sequential_serial"].tokens
    for name, r in results.items():
        if name not in FUSED:
            assert r.tokens == base, name


@pytest.mark.parametrize("run", ["pipelined_P2_split", "mixed_fused_chunks"])
def test_tokens_match_oracle_teacher_forced(results, run):
    d = M.TINY
    o = M.OracleModel(d)
    toks = results[run].tokens
    bad = []
    for rid in range(8):
        prompt = M.prompt_tokens(d.seed, rid, 64, d.vocab)
        row = list(range(100 * rid, 100 * rid + 8))
        lg = o.prefill([prompt], [row])[0]
        seq = toks[rid]
        for g in range(32):
            tol = 1e-2 * float(np.max(np.abs(lg)))
            if M.top2_margin(lg) > tol and int(np.argmax(lg)) != seq[g]:
                bad.append((rid, g))
            if g + 1 < 32:
                lg = o.decode([seq[g]], [64 + g], [row])[0]
        o.release(row)
    assert not bad, bad


def test_page_tables_bit_exact(results):
    from paper_2505_03763_b200.runtime import parse_devpages

    for name, r in results.items():
        dev = parse_devpages(r)
        assert dev == r.pages, name
        assert P.page_replay(r.journal, 480) == r.pages, name
        # each request held blocks_for(in + out) pages at its largest extent
        assert all(len(v) == P.blocks_for(64 + 32) for v in r.pages.values()), name


def test_event_log_contract(results):
    for name, r in results.items():
        for t, inst, logged, replayed in P.ledger_replay(r.event_log):
            assert logged == replayed, (name, t)
        assert all(q["ttft_s"] > 0 and q["e2e_s"] >= q["ttft_s"] for q in r.requests), name


def test_green_partition_reported(results):
    for name in ("pipelined_P2_green48", "mixed_green64_arrivals"):
        gpu = {}
        for line in results[name].text.splitlines():
            if line.startswith("#gpu "):
                gpu = dict(kv.split("=") for kv in line[5:].split(";"))
        want = 48 if "48" in name else 64
        assert int(gpu["decode_sms"]) == want, (name, gpu)
        assert int(gpu["decode_sms"]) + int(gpu["prefill_sms"]) == 148 or int(gpu["prefill_sms"]) > 0, gpu


def test_fused_run_used_mixed_launches(results):
    gpu = {}
    for line in results["mixed_fused_chunks"].text.splitlines():
        if line.startswith("#gpu "):
            gpu = dict(kv.split("=") for kv in line[5:].split(";"))
    assert gpu["fuse"] == "1" and int(gpu["mixed_launches"]) > 0, gpu

"""Scheduler/ledger/log/metrics parity against the compiled reference.

The product's virtual-clock backend (sw_sim_run) and the UNMODIFIED reference
simulator (oracle/_ref/refsim, built from /root/reference/proj/include) are run
on the same spec; the event-log CSV (engine.hpp semantics, event_log.hpp
encoding), the report scalars (metrics.hpp) and the per-request rows must be
byte-identical.  Cases mirror the reference's property generator
(tests/property_core.hpp:26-87) minus the time-sliced discipline (out of
scope), plus the shipped experiment configs (configs/*.json).
"""
import random

import pytest

from conftest import refsim


def _strip_pages(text: str) -> str:
    return "".join(l + "\n" for l in text.splitlines() if not l.startswith(("#pages", "#journal")))


def _compare(swlib, spec: str):
    code, ref_out, ref_err = refsim(spec)
    if code != 0:
        with pytest.raises(swlib.SplitwiseError) as ei:
            swlib.sim_run(spec)
        kind = {2: swlib.ConfigError, 4: swlib.ContractViolation}[code]
        assert isinstance(ei.value, kind), (spec, ref_err, str(ei.value))
        return None
    mine = swlib.sim_run(spec)
    assert _strip_pages(mine.text) == ref_out, spec
    return mine


def random_spec(seed: int) -> str:
    r = random.Random(seed)
    n = r.randint(0, 10)
    in_lo = r.randint(1, 48)
    out_lo = r.randint(1, 6)
    spec = {
        "n": n,
        "input": f"{in_lo}..{in_lo + r.randint(0, 16)}",
        "output": f"{out_lo}..{out_lo + r.randint(0, 2)}",
        "seed": r.getrandbits(63),
        "arrival": r.choice(["zero", f"fixed:{0.001 * r.randint(0, 5)}", "poisson:200"]),
        "max_batch": r.randint(0, 4),
    }
    pol = r.choice(["sequential", "pipelined_splitwiser", "continuous_batching", "mixed_batching", "multi_instance"])
    spec["policy"] = pol
    n_inst = 1
    if pol == "pipelined_splitwiser":
        n_inst = spec["P"] = r.randint(1, 3)
    elif pol == "multi_instance":
        n_inst = spec["n_instances"] = r.randint(2, 3)
        spec["inner"] = r.choice(["sequential", "continuous_batching", "mixed_batching"])
    max_fp = 1 + (in_lo + 16 + out_lo + 2) // 16
    spec["kv_capacity_blocks"] = n_inst * (max_fp + r.randint(0, 50))
    spec["mode"] = "mps_concurrent" if n_inst > 1 else r.choice(["exclusive", "mps_concurrent"])
    if r.random() < 0.2:
        spec["cost.kv_handoff_s"] = 0.0005
    return ";".join(f"{k}={v}" for k, v in spec.items())


@pytest.mark.parametrize("seed", range(300))
def test_random_case_matches_reference(swlib, seed):
    _compare(swlib, random_spec(seed))


SHIPPED = {
    # configs/*.json of the reference, as specs
    "vllm_sp": "n=160;input=1024;output=1024;seed=1;policy=continuous_batching;max_batch=0;mode=exclusive",
    "vllm_mpsx2": "n=160;input=1024;output=1024;seed=1;policy=multi_instance;n_instances=2;"
                  "inner=continuous_batching;mode=mps_concurrent",
    "hf_sequential": "n=160;input=512;output=20;seed=1;policy=sequential;max_batch=20;mode=exclusive",
    "hf_splitwiser_P8": "n=160;input=512;output=20;seed=1;policy=pipelined_splitwiser;P=8;max_batch=20;"
                        "mode=mps_concurrent",
    "mixed_poisson": "n=64;input=128..2048;output=256;seed=1;arrival=poisson:40;policy=mixed_batching;"
                     "mode=exclusive",
}


@pytest.mark.parametrize("name", sorted(SHIPPED))
def test_shipped_configs_match_reference(swlib, name):
    _compare(swlib, SHIPPED[name])


def test_capacity_and_contract_errors_match(swlib):
    # request larger than the instance: ContractViolation in both
    _compare(swlib, "n=2;input=1024;output=8;policy=continuous_batching;kv_capacity_blocks=10")
    # exclusive with several instances: ConfigError in both
    _compare(swlib, "n=2;input=16;output=2;policy=multi_instance;n_instances=2;mode=exclusive")


TRACE = """id,arrival_s,input_tokens,output_tokens
3,0.0,300,12
0,0.0,64,4
7,0.0015,900,30
1,0.002,128,1
5,0.002,2048,8
2,0.0105,17,40
"""


@pytest.mark.parametrize("policy", ["policy=continuous_batching", "policy=mixed_batching;max_batch=2",
                                    "policy=pipelined_splitwiser;P=2;max_batch=3;mode=mps_concurrent",
                                    "policy=sequential;max_batch=4"])
def test_trace_workload_matches_reference(swlib, tmp_path, policy):
    """workload.trace (config.hpp assemble + request.hpp parse_trace): sorted by arrival, ties by id."""
    p = tmp_path / "trace.csv"
    p.write_text(TRACE)
    _compare(swlib, f"trace={p};{policy}")


def test_trace_errors_match_reference(swlib, tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("id,arrival_s,input_tokens,output_tokens\n1,0.0,10,2\n1,0.5,10,2\n")  # duplicate id
    _compare(swlib, f"trace={bad};policy=continuous_batching")
    _compare(swlib, f"trace={tmp_path / 'missing.csv'};policy=continuous_batching")

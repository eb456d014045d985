"""C-ABI surface (CPU): the library loads, exports every symbol of
include/splitwise.h, maps the reference error taxonomy onto status codes, and
the spec front end derives KV capacity like config.hpp:66-79."""
import re
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "splitwise.h")).read()
    return sorted(set(re.findall(r"\b(sw_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(swlib):
    L = swlib.lib()
    declared = declared_symbols()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(swlib.EXPORTED_SYMBOLS) <= set(declared)


def test_error_taxonomy(swlib):
    with pytest.raises(swlib.ConfigError):
        swlib.sim_run("n=2;input=4;output=1;policy=nonsense")
    with pytest.raises(swlib.ConfigError):
        swlib.sim_run("n=2;input=4;output=1;bogus_key=1")
    with pytest.raises(swlib.ConfigError):
        swlib.sim_run("n=2;input=5..4;output=1")  # min > max
    with pytest.raises(swlib.ContractViolation):
        swlib.sim_run("n=1;input=1024;output=8;policy=continuous_batching;kv_capacity_blocks=10")
    assert "ContractViolation" in swlib.lib().sw_last_error().decode()


# The reference's own weight-accounting golden (tests/test_config.cpp:101-113):
# budget 2e4, unit 1, weights 5e3 -> shared 15000, duplicated over 2 instances
# 10000, single instance 15000, explicit override 777.
GOLDEN_KV = [
    ("policy=multi_instance;n_instances=2;mode=mps_concurrent;shared_weights=true", "7500|7500"),
    ("policy=multi_instance;n_instances=2;mode=mps_concurrent;shared_weights=false", "5000|5000"),
    ("policy=continuous_batching;shared_weights=false", "15000"),
    ("policy=multi_instance;n_instances=2;mode=mps_concurrent;shared_weights=false;kv_capacity_blocks=777", "389|388"),
]


@pytest.mark.parametrize("extra,expect", GOLDEN_KV)
def test_kv_capacity_derivation_golden(swlib, extra, expect):
    r = swlib.sim_run(f"n=2;input=16;output=1;mem_budget_units=20000;block_mem_unit=1;weight_mem_units=5000;{extra}")
    meta = r.event_log.splitlines()[1]
    assert f"kv_capacity={expect};" in meta


def test_duplicated_weights_shrink_capacity(swlib):
    # P=2 splitwiser lanes with private weight copies: one extra copy of 16 units
    r = swlib.sim_run("n=2;input=16;output=1;policy=pipelined_splitwiser;P=2;mode=mps_concurrent;"
                      "shared_weights=false;mem_budget_units=1016;weight_mem_units=16")
    meta = r.event_log.splitlines()[1]
    assert "kv_capacity=492|492;" in meta  # (1016-16-16) = 984 split over 2 instances


def test_page_journal_replays_to_page_rows(swlib):
    from oracle import pages as P

    r = swlib.sim_run("n=12;input=20..70;output=1..9;seed=5;arrival=poisson:300;policy=mixed_batching;"
                      "max_batch=4;kv_capacity_blocks=64")
    assert P.page_replay(r.journal, 64) == r.pages
    for t, inst, logged, replayed in P.ledger_replay(r.event_log):
        assert logged == replayed

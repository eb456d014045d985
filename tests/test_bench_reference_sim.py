"""bench.py's `reference_simulator` leg: the unmodified reference simulator
(oracle/_ref/refsim) run on the bench workloads' traces and policies.  Its
simulated report must equal the product's virtual-clock drop-in (sw_sim_run)
on the same spec -- the bench line's reference prediction is the reference's
own number, not a re-computation."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REFSIM = os.path.join(ROOT, "oracle", "_ref", "refsim")
pytestmark = pytest.mark.skipif(not os.access(REFSIM, os.X_OK), reason="oracle/_ref/refsim not built")


@pytest.mark.parametrize("name", ["8b-cfg3", "1b", "8b-long", "tiny"])
def test_reference_simulator_matches_sim_run(name):
    import bench
    import paper_2505_03763_b200 as sw

    w = dict(bench.WORKLOADS[name])
    in_max = int(str(w["input"]).split("..")[-1])
    pages = w["n"] * ((in_max + w["output"] + 15) // 16) + 64
    r = bench.reference_simulator(w, pages)
    assert r is not None and "error" not in r, r
    for arm in ("split", "serial"):
        spec = (f"n={w['n']};input={w['input']};output={w['output']};seed=1;arrival={w['arrival']};"
                f"kv_capacity_blocks={pages};{r[arm]['policy']}")
        if "mode=time_sliced" in spec:
            # the time-sliced law models OS time slicing of separate processes: out of scope here
            with pytest.raises(sw.ConfigError):
                sw.sim_run(spec)
            continue
        ours = sw.sim_run(spec)
        assert round(float(ours.report["tokens_per_s"]), 1) == r[arm]["simulated_tokens_per_s"]
    assert r["simulated_split_over_serial"] > 0


def test_weak_scaling_keeps_the_per_gpu_rate():
    """bench.spec_for at N ranks: n * N requests at N times the rate, so each
    round-robin shard is the single-GPU workload (512 requests over ~4 s on
    configs[2]), not an N-times thinner arrival-bound stream."""
    import bench
    import paper_2505_03763_b200 as sw

    assert bench.global_arrival("poisson:128", 1) == "poisson:128"
    assert bench.global_arrival("poisson:128", 4) == "poisson:512"
    assert bench.global_arrival("fixed:0.02", 2) == "fixed:0.01"
    assert bench.global_arrival("zero", 8) == "zero"
    w = dict(bench.WORKLOADS["8b-cfg3"], kv_pages=73792)

    def arrivals(rank, world):
        r = sw.sim_run(bench.spec_for(w, "policy=continuous_batching;max_batch=256", rank, world))
        return [float(l.split(",", 1)[0]) for l in r.event_log.splitlines() if ",arrival," in l]

    one = arrivals(0, 1)
    for world in (2, 4, 8):
        shard = arrivals(world - 1, world)
        assert len(shard) == len(one) == 512
        assert abs(shard[-1] - one[-1]) / one[-1] < 0.25, (world, shard[-1], one[-1])

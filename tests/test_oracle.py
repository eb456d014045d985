"""The oracle itself, pinned before it is trusted (CPU only).

* SplitMix64 against the compiled reference (oracle/_ref/refsim --prng) and the
  reference's frozen Poisson golden (tests/test_util.hpp:18, test_workload.cpp:76-93);
* the C weight generator (oracle/gen.c) against the numpy restatement;
* self-consistency of the paged-KV decoder: the prompt pass's last-position
  logits equal a decode step that feeds the last prompt token after a prompt
  pass over the first n-1 tokens (same pages, different page order).
"""
import subprocess

import numpy as np
import pytest

from conftest import REFSIM, refsim
from oracle import model as M

K_POISSON_GOLDEN_MEAN = 0.24759804680176598  # reference tests/test_util.hpp:18


def test_splitmix_matches_reference():
    import os

    if not os.path.exists(REFSIM):
        pytest.skip("refsim not built")
    for seed in (0, 1, 12345, 2**63 + 17):
        ref = [int(x) for x in subprocess.run([REFSIM, "--prng", str(seed), "50"], capture_output=True,
                                              text=True).stdout.split()]
        assert ref == M.next_u64_stream(seed, 50)


def test_poisson_golden_mean_through_product(swlib):
    r = swlib.sim_run("n=10000;input=1;output=1;seed=7;arrival=poisson:4;policy=continuous_batching")
    arr = sorted(q["arrival_s"] for q in r.requests)
    gaps = np.diff([0.0] + arr)
    assert abs(gaps.mean() - K_POISSON_GOLDEN_MEAN) < 1e-12


def test_c_generator_matches_numpy():
    gen = M._c_gen()
    if not gen:
        pytest.skip("oracle/_build/libgen.so not built")
    for k, rows, cols, fan in [(0, 97, 64, 64), (5, 300, 256, 256), (17, 64, 2048, 8192)]:
        a = M.tensor_values(3, k, rows, cols, fan, use_c=True)
        b = M.tensor_values(3, k, rows, cols, fan, use_c=False)
        assert np.array_equal(a, b)


def test_weights_are_bf16_valued_and_scaled():
    w = M.tensor_values(1, 3, 256, 256, 256, use_c=False)
    assert np.array_equal(M.bf16_round(w), w)
    bound = np.sqrt(3.0 / 256)
    assert np.abs(w).max() <= bound * 1.01 and abs(w.std() - bound / np.sqrt(3)) < 0.01 * bound


@pytest.mark.parametrize("emulate", [False, True])
def test_oracle_prefill_equals_incremental_decode(emulate):
    d = M.TINY
    o = M.OracleModel(d, emulate_bf16=emulate)
    p = M.prompt_tokens(d.seed, 3, 37, d.vocab)
    full = o.prefill([p], [[5, 6, 7]])[0]
    o2 = M.OracleModel(d, emulate_bf16=emulate, share_weights_with=o)
    o2.prefill([p[:-1]], [[9, 2, 4]])
    step = o2.decode([int(p[-1])], [len(p) - 1], [[9, 2, 4]])[0]
    tol = 1e-5 if not emulate else 2e-2  # emulation rounds P differently in the two phases
    assert np.linalg.norm(full - step) / np.linalg.norm(full) < tol


def test_prompt_tokens_in_range_and_deterministic():
    a = M.prompt_tokens(1, 7, 1000, 128256)
    assert a.min() >= 0 and a.max() < 128256
    assert np.array_equal(a, M.prompt_tokens(1, 7, 1000, 128256))
    assert not np.array_equal(a, M.prompt_tokens(1, 8, 1000, 128256))

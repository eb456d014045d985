"""Regenerate the committed golden fixtures (TEST INFRASTRUCTURE ONLY).

Run here, where /root/reference exists:  python tests/golden/make_golden.py

* sched_golden.json -- (files:*) sha256 of the reference's experiment files
  (oracle/_ref/refwrite: write_experiment) for 6 randomized specs; and
  the UNMODIFIED reference simulator (oracle/_ref/refsim,
  compiled from /root/reference/proj/include by oracle/Makefile) run on the
  shipped configs (configs/*.json as specs) and on 40 randomized specs from
  tests/test_sched_parity.random_spec.  Small outputs are stored verbatim,
  large ones as sha256 + their report block.  The GPU box has no
  /root/reference; these fixtures let the product's scheduler path be checked
  there (and here without rebuilding refsim).
* tiny_cfg1.npz -- BASELINE configs[0] through the fp32 oracle (oracle/model.py):
  8 prompts x 64 tokens (SplitMix64 prompts, seed 1), 32 greedy steps each
  (serial generate_greedy).  Frozen on first generation like the reference's
  kPoissonGoldenMean (tests/test_util.hpp:18); the model math has no reference
  implementation, so this pins our oracle across machines and
  gives the GPU tests a fixed target.
"""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import model as M  # noqa: E402

REFSIM = os.path.join(ROOT, "oracle", "_ref", "refsim")
VERBATIM_LIMIT = 24 * 1024
N_RANDOM = 40


def report_block(text: str) -> str:
    """The report scalars (lines after the event-log CSV), kept verbatim for large runs."""
    lines = text.splitlines()
    return "\n".join(l for l in lines if l.startswith("#report"))


def sched_cases():
    from test_sched_parity import SHIPPED, random_spec

    cases = {f"shipped:{k}": v for k, v in sorted(SHIPPED.items())}
    for s in range(N_RANDOM):
        cases[f"random:{s}"] = random_spec(1000 + s)
    return cases


def random_spec_files(s):
    from test_sched_parity import random_spec

    return random_spec(3000 + s)


def make_sched():
    out = {}
    for name, spec in sched_cases().items():
        p = subprocess.run([REFSIM, spec], capture_output=True, text=True)
        rec = {"spec": spec, "code": p.returncode, "sha256": hashlib.sha256(p.stdout.encode()).hexdigest(),
               "bytes": len(p.stdout)}
        if p.returncode == 0 and len(p.stdout) <= VERBATIM_LIMIT:
            rec["stdout"] = p.stdout
        elif p.returncode == 0:
            rec["report"] = report_block(p.stdout)
        out[name] = rec
    # the reference's experiment files (write_experiment) for a few specs: sha256 per file
    import tempfile
    refwrite = os.path.join(ROOT, "oracle", "_ref", "refwrite")
    for i, spec in enumerate([random_spec_files(s) for s in range(6)]):
        d = tempfile.mkdtemp()
        p = subprocess.run([refwrite, "--write", d, spec], capture_output=True, text=True)
        if p.returncode != 0:
            continue
        out[f"files:{i}"] = {"spec": spec, "sha256": {
            f: hashlib.sha256(open(os.path.join(d, f)).read().encode()).hexdigest()
            for f in ("report.json", "requests.csv", "timeseries.csv", "events.csv")}}
    with open(os.path.join(HERE, "sched_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(f"sched_golden.json: {len(out)} cases")


def make_tiny():
    d = M.TINY
    o = M.OracleModel(d)
    n_req, n_in, n_out = 8, 64, 32
    prompts = np.stack([M.prompt_tokens(d.seed, r, n_in, d.vocab) for r in range(n_req)]).astype(np.int32)
    toks, margins, first_logits, last_logits = [], [], [], []
    for r in range(n_req):
        row = list(range(r * 8, r * 8 + 8))  # 8 pages of 16 = 128 >= 64 + 32 positions
        t, lg = M.generate_greedy(o, prompts[r], n_out, row)
        o.release(row)
        toks.append(t)
        lg = np.stack(lg)
        margins.append(M.top2_margin(lg) / np.abs(lg).max(axis=1))
        first_logits.append(lg[0])
        last_logits.append(lg[-1])
    np.savez_compressed(os.path.join(HERE, "tiny_cfg1.npz"), prompts=prompts, tokens=np.array(toks, np.int32),
                        rel_margin=np.array(margins, np.float32), first_logits=np.array(first_logits, np.float32),
                        last_logits=np.array(last_logits, np.float32))
    print("tiny_cfg1.npz written")


if __name__ == "__main__":
    if not os.path.exists(REFSIM):
        sys.exit("oracle/_ref/refsim missing: run `make -C oracle` where /root/reference exists")
    make_sched()
    make_tiny()

"""Repeat one GPU engine run until the KV ledger replay disagrees with a logged kv record;
print the event log around the first mismatch (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import model as M
from oracle import pages as P
from paper_2505_03763_b200 import runtime

SPEC = ("n=8;input=64;output=32;seed=1;kv_capacity_blocks=480;policy=mixed_batching;arrival=fixed:0.0005;"
        "engine.split=1;engine.fuse=1;engine.chunk_tokens=96")
eng = runtime.Engine(M.TINY, max_prefill_tokens=1024, max_decode_batch=16, n_pages=512, n_slots=16,
                     max_pages_per_slot=8, max_out=40)
for it in range(40):
    r = eng.run(SPEC)
    bad = [(t, l, rp) for t, inst, l, rp in P.ledger_replay(r.event_log) if l != rp]
    if bad:
        t0 = bad[0][0]
        print(f"run {it}: first mismatch at t={t0}: logged {bad[0][1]} replayed {bad[0][2]}")
        lines = r.event_log.splitlines()
        idx = [i for i, ln in enumerate(lines) if ln.startswith(repr(t0)[:8]) or ln.split(",")[0] == str(t0)]
        for ln in lines:
            if ln.split(",")[1] in ("meta",):
                continue
            try:
                tt = float(ln.split(",")[0])
            except ValueError:
                print(ln)
                continue
            if abs(tt - t0) < 0.0012:
                print(ln)
        break
else:
    print("no mismatch in 40 runs")
eng.close()

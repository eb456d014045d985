"""Engine runs for compute-sanitizer (racecheck / synccheck / memcheck): the TINY
model through sw_engine_run under the co-scheduling modes that put two streams
on one KV arena -- split streams (mixed batching), fused mixed steps, chunked
prefill (chunks reading the cached prefix), green-context partitions.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_03763_b200 import runtime, shapes

SPECS = [
    "policy=mixed_batching;max_batch=4;engine.split=1",
    "policy=mixed_batching;max_batch=4;engine.split=1;engine.fuse=1",
    "policy=chunked_prefill;max_batch=4;chunk_tokens=128;engine.split=1;engine.fuse=1",
    "policy=pipelined_splitwiser;P=2;max_batch=2;engine.split=1;engine.decode_sms=48",
]


def main():
    eng = runtime.Engine(shapes.TINY, max_prefill_tokens=1024, max_decode_batch=8, n_pages=256, n_slots=16,
                         max_pages_per_slot=16, max_out=16)
    for s in SPECS:
        r = eng.run(f"n=6;input=60..200;output=4..8;seed=3;arrival=poisson:500;kv_capacity_blocks=256;{s}")
        print(f"ok {r.report['total_output_tokens']} tokens | {s}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

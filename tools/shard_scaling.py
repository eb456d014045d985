"""Request-sharded scaling projected shard by shard on one B200.

The multi-GPU path has no data-path collective: rank r of N runs its own engine
on its round-robin shard of the global trace (bench.spec_for: `shard=r/N`, the
reference's multi_instance_split, with the per-GPU arrival rate kept) and the
ranks meet once, after the run, to gather request rows.  What GPU r does is
therefore exactly one engine run of shard r, so this tool runs every shard of
N in {1, 2, 4, 8} on the one GPU it has, one after another, and folds them as
bench.py would: aggregate tokens/s = sum of tokens / max shard makespan, p50s
over the union of request rows.  Not captured: host-CPU contention between
ranks sharing a node and the end-of-run gather (one all_gather of ~1 MB per rank).

  python tools/shard_scaling.py [--workload 8b-cfg3] [--ns 1,2,4,8] [--arm split|serial|both]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench
from paper_2505_03763_b200 import runtime, shapes, sharded


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="8b-cfg3")
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--arm", default="both")
    args = ap.parse_args()
    w = dict(bench.WORKLOADS[args.workload])
    desc = getattr(shapes, w["model"])
    in_max = int(str(w["input"]).split("..")[-1])
    pages_per = (in_max + w["output"] + 15) // 16
    eng = runtime.Engine(desc, max_prefill_tokens=w["max_prefill"], max_decode_batch=w["max_decode"], n_pages=None,
                         n_slots=w["n"] + 8, max_pages_per_slot=pages_per + 1, max_out=w["output"] + 1,
                         kv_reserve_bytes=4 << 30, max_pages=w["n"] * pages_per + 64)
    w["kv_pages"] = eng.n_pages
    arms = ["split", "serial"] if args.arm == "both" else [args.arm]
    for arm in arms:
        eng.run(bench.spec_for(w, w[arm], 0, 1))  # warm (graphs, attributes)
    base = {}
    for arm in arms:
        for n in [int(x) for x in args.ns.split(",")]:
            rows, shards = [], []
            for r in range(n):
                t0 = time.perf_counter()
                res = eng.run(bench.spec_for(w, w[arm], r, n))
                wall = time.perf_counter() - t0
                mk = res.report["makespan_s"]
                shards.append({"rank": r, "makespan_s": round(mk, 4), "tokens": int(res.report["total_output_tokens"]),
                               "wall_s": round(wall, 2)})
                rows += sharded.request_rows(res)
            mk = max(s["makespan_s"] for s in shards)
            f = sharded.fold(sorted(rows, key=lambda q: q["id"]), mk)
            agg = f["total_output_tokens"] / mk
            if n == 1:
                base[arm] = agg
            line = {"workload": args.workload, "arm": arm, "n_gpus": n, "policy": w[arm],
                    "arrival_global": bench.global_arrival(w["arrival"], n), "requests": f["n_requests"],
                    "aggregate_tokens_per_s": round(agg, 1), "per_gpu_tokens_per_s": round(agg / n, 1),
                    "efficiency_vs_n1": round(agg / (n * base[arm]), 4) if arm in base else None,
                    "p50_ttft_s": round(f["p50_ttft_s"], 4), "p50_tbt_s": round(f["p50_tbt_s"], 5),
                    "shard_makespans_s": [s["makespan_s"] for s in shards]}
            print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()

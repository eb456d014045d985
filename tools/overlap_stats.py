"""Phase-overlap statistics of GPU engine runs from their event logs (device
timestamps): how long prompt tasks and token steps take alone vs while the
other phase is in flight, and how much of the makespan has both phases active.

  python tools/overlap_stats.py [--workload 1b] [--specs "policy=...;engine.split=1" ...]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402  (workload table)


def parse(text):
    tasks = {}
    for line in text.splitlines():
        if line.startswith("#") or line.startswith("time_s"):
            continue
        t, kind, detail = line.split(",", 2)
        kv = dict(x.split("=", 1) for x in detail.split(";") if "=" in x)
        if kind == "task_start":
            tasks[int(kv["task"])] = {"kind": kv["kind"], "start": float(t), "batch": kv.get("batch")}
        elif kind == "task_complete":
            tasks[int(kv["task"])]["end"] = float(t)
    return [v for v in tasks.values() if "end" in v]


def overlap(a, others):
    return sum(max(0.0, min(a["end"], o["end"]) - max(a["start"], o["start"])) for o in others)


def stats(tasks):
    pro = [t for t in tasks if t["kind"] == "prompt"]
    tok = [t for t in tasks if t["kind"] != "prompt"]
    out = {}
    for name, group, other in (("prompt", pro, tok), ("token_step", tok, pro)):
        alone = [t["end"] - t["start"] for t in group if overlap(t, other) == 0]
        shared = [t["end"] - t["start"] for t in group if overlap(t, other) > 0]
        out[name] = (len(group), sum(alone) / max(1, len(alone)), len(alone), sum(shared) / max(1, len(shared)),
                     len(shared))
    # wall time with both phases active
    ev = sorted([(t["start"], 1 if t["kind"] == "prompt" else 2, +1) for t in tasks] +
                [(t["end"], 1 if t["kind"] == "prompt" else 2, -1) for t in tasks])
    act = {1: 0, 2: 0}
    last = ev[0][0] if ev else 0.0
    both = busy = 0.0
    for t, k, d in ev:
        if act[1] and act[2]:
            both += t - last
        if act[1] or act[2]:
            busy += t - last
        act[k] += d
        last = t
    out["both_active_s"] = both
    out["busy_s"] = busy
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="1b")
    ap.add_argument("--specs", nargs="*", default=None)
    args = ap.parse_args()
    from oracle import model as M
    from paper_2505_03763_b200 import runtime

    w = dict(bench.WORKLOADS[args.workload])
    desc = getattr(M, w["model"])
    in_max = int(str(w["input"]).split("..")[-1])
    pages_per = (in_max + w["output"] + 15) // 16
    w["kv_pages"] = w["n"] * pages_per + 64
    eng = runtime.Engine(desc, max_prefill_tokens=w["max_prefill"], max_decode_batch=w["max_decode"],
                         n_pages=w["kv_pages"], n_slots=w["n"] + 8, max_pages_per_slot=pages_per + 1,
                         max_out=w["output"] + 1)
    specs = args.specs or [w["split"], w["serial"], w["best_serial"]]
    for extra in specs:
        spec = bench.spec_for(w, extra, 0, 1)
        for _ in range(2):
            eng.run(spec)  # warm (graphs, attributes)
        r = eng.run(spec)
        s = stats(parse(r.text))
        print(f"== {extra}")
        print(f"   makespan {r.report['makespan_s'] * 1e3:.1f} ms, tokens/s {r.report['tokens_per_s']:.0f}, "
              f"both phases active {s['both_active_s'] * 1e3:.1f} ms of {s['busy_s'] * 1e3:.1f} ms busy")
        for name in ("prompt", "token_step"):
            n, a, na, sh, ns = s[name]
            print(f"   {name:10s} n={n:4d}  alone {a * 1e3:8.3f} ms (x{na})  while other phase runs "
                  f"{sh * 1e3:8.3f} ms (x{ns})")
    eng.close()


if __name__ == "__main__":
    main()

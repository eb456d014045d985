"""Request-sharded scale-out: every GPU runs its own split
engine on its round-robin share of one trace (spec key `shard=r/N`, the
reference's multi_instance_split routing, splitsim/schedulers.hpp:86-92), and
the only collective is one gather of the per-request results at the end of the
run, folded into global metrics exactly as the reference folds one run
(splitsim/metrics.hpp:79-85 nearest_rank, :317-362 the per-request folds).

`gather_requests` is backend-agnostic torch.distributed (NCCL over NVLink on
the GPU box, gloo in the CPU tests): each rank packs a fixed-size float64
block {request id, arrival, TTFT, E2E, mean TBT, tokens, token ids...} so one
all_gather moves it (a few MB at 8B cfg4 scale, off the critical path)."""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

FIELDS = ("id", "arrival_s", "ttft_s", "e2e_s", "tbt_mean_s", "n_tokens", "n_ids")


def nearest_rank(sorted_vals: Sequence[float], q: float) -> float:
    """The reference's percentile rule (metrics.hpp:79-85; csrc/host/report.hpp nearest_rank)."""
    n = len(sorted_vals)
    if n == 0:
        return 0.0
    idx = min(max(int(math.ceil(q * n)), 1), n)
    return sorted_vals[idx - 1]


def request_rows(res) -> List[Dict[str, object]]:
    """Per-request rows of one RunResult: the `#request` metrics, the output
    token count from the request's arrival record, and the generated token ids
    (`#tokens`, GPU runs only)."""
    outputs = {}
    for line in res.event_log.splitlines():
        if ",arrival," in line:
            kv = dict(x.split("=", 1) for x in line.split(",", 2)[2].split(";") if "=" in x)
            outputs[int(kv["req"])] = int(kv["output"])
    rows = []
    for q in res.requests:
        rid = int(q["id"])
        toks = list(res.tokens.get(rid, []))
        rows.append({"id": rid, "arrival_s": q["arrival_s"], "ttft_s": q["ttft_s"], "e2e_s": q["e2e_s"],
                     "tbt_mean_s": q["tbt_mean_s"], "n_tokens": outputs[rid], "n_ids": len(toks), "tokens": toks})
    return rows


def fold(rows: Sequence[Dict[str, object]], makespan_s: float) -> Dict[str, float]:
    """Global metrics over every rank's requests: the same folds as one run's
    report (TTFT over all requests; TBT over the per-request means of requests
    with more than one token, metrics.hpp:317-362)."""
    ttft = sorted(float(r["ttft_s"]) for r in rows)
    tbt = sorted(float(r["tbt_mean_s"]) for r in rows if int(r["n_tokens"]) > 1 and not math.isnan(float(r["tbt_mean_s"])))
    e2e = sorted(float(r["e2e_s"]) for r in rows)
    tokens = sum(int(r["n_tokens"]) for r in rows)
    return {"n_requests": len(rows), "total_output_tokens": tokens, "makespan_s": makespan_s,
            "tokens_per_s": tokens / makespan_s if makespan_s > 0 else 0.0,
            "p50_ttft_s": nearest_rank(ttft, 0.5), "p99_ttft_s": nearest_rank(ttft, 0.99),
            "p50_tbt_s": nearest_rank(tbt, 0.5) if tbt else float("nan"),
            "p99_tbt_s": nearest_rank(tbt, 0.99) if tbt else float("nan"),
            "median_e2e_s": nearest_rank(e2e, 0.5)}


def gather_requests(dist, world: int, rows: Sequence[Dict[str, object]], makespan_s: float, wall_s: float,
                    device, max_requests: int, max_tokens: int):
    """All-gather every rank's request rows (one collective).  Returns
    (all rows sorted by id, max makespan over ranks, max wall over ranks)."""
    import torch

    if len(rows) > max_requests:
        raise ValueError(f"gather_requests: {len(rows)} rows > max_requests {max_requests}")
    width = len(FIELDS) + max_tokens
    buf = torch.full((max_requests + 1, width), -1.0, dtype=torch.float64)
    buf[0, 0], buf[0, 1], buf[0, 2] = float(len(rows)), float(makespan_s), float(wall_s)
    for i, r in enumerate(rows):
        toks = list(r["tokens"])
        if len(toks) > max_tokens:
            raise ValueError(f"gather_requests: request {r['id']} has {len(toks)} tokens > max_tokens {max_tokens}")
        buf[i + 1, :len(FIELDS)] = torch.tensor([float(r[f]) for f in FIELDS], dtype=torch.float64)
        if toks:
            buf[i + 1, len(FIELDS):len(FIELDS) + len(toks)] = torch.tensor(toks, dtype=torch.float64)
    buf = buf.to(device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    all_rows, makespan, wall = [], 0.0, 0.0
    for b in out:
        b = b.cpu()
        n = int(b[0, 0])
        makespan, wall = max(makespan, float(b[0, 1])), max(wall, float(b[0, 2]))
        for i in range(n):
            v = b[i + 1]
            row = {f: float(v[j]) for j, f in enumerate(FIELDS)}
            row["id"], row["n_tokens"], row["n_ids"] = int(row["id"]), int(row["n_tokens"]), int(row["n_ids"])
            row["tokens"] = [int(x) for x in v[len(FIELDS):len(FIELDS) + row["n_ids"]]]
            all_rows.append(row)
    all_rows.sort(key=lambda r: r["id"])
    return all_rows, makespan, wall

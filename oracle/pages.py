"""ORACLE / TEST INFRASTRUCTURE ONLY -- independent replay of the KV ledger.

Two restatements used to check the product's KV bookkeeping:

* `ledger_replay(event_log_csv)` recomputes every instance's block total from
  the record stream alone, exactly like the reference's KV conservation oracle
  (tests/property_core.hpp:97-145): a prompt adds blocks_for(input) per
  request, token step g adds blocks_for(in+g) - blocks_for(in+g-1) and the
  final step frees blocks_for(in+out-1).  Every `kv` record must match.
* `page_replay(journal, n_pages)` replays the physical alloc/free journal
  through a lowest-free-id-first allocator (the policy csrc/host/kv.hpp
  documents) and returns each request's page-table row at its largest extent,
  which must equal the GPU's page table bit for bit.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Tuple


def blocks_for(tokens: int, block_tokens: int = 16) -> int:
    return (tokens + block_tokens - 1) // block_tokens


def ledger_replay(csv: str) -> List[Tuple[float, int, int, int]]:
    """Returns [(time, instance, logged_blocks, replayed_blocks)] for every kv record."""
    req = {}
    gen = {}
    inst_of = {}
    batches = {}
    task = {}
    totals: Dict[int, int] = {}
    B = 16
    out = []
    for line in csv.splitlines()[1:]:
        t, kind, detail = line.split(",", 2)
        kv = dict(item.split("=", 1) for item in detail.split(";") if item)
        if kind == "meta":
            B = int(kv["block_tokens"])
        elif kind == "batch_def":
            batches[int(kv["batch"])] = [int(x) for x in kv["reqs"].split("|") if x]
        elif kind == "arrival":
            req[int(kv["req"])] = (int(kv["input"]), int(kv["output"]))
            gen[int(kv["req"])] = 0
        elif kind == "task_start":
            task[int(kv["task"])] = (kv["kind"], int(kv["batch"]))
            if kv["kind"] == "prompt":
                inst = int(kv["inst"])
                for rid in batches[int(kv["batch"])]:
                    if rid in inst_of:  # a later chunk of a chunked prompt: allocated by its first chunk
                        continue
                    totals[inst] = totals.get(inst, 0) + blocks_for(req[rid][0], B)
                    inst_of[rid] = inst
        elif kind == "task_complete":
            k, b = task[int(kv["task"])]
            if k != "token_step":
                continue
            for rid in batches[b]:
                i, o = req[rid]
                gen[rid] += 1
                g = gen[rid]
                inst = inst_of[rid]
                if g == o:
                    totals[inst] -= blocks_for(i + g - 1, B)
                else:
                    totals[inst] += blocks_for(i + g, B) - blocks_for(i + g - 1, B)
        elif kind == "kv":
            inst = int(kv["inst"])
            out.append((float(t), inst, int(kv["blocks"]), totals.get(inst, 0)))
    return out


def page_replay(journal: List[Tuple[int, int]], n_pages: int) -> Dict[int, List[int]]:
    free = list(range(n_pages))
    heapq.heapify(free)
    rows: Dict[int, List[int]] = {}
    final: Dict[int, List[int]] = {}
    for rid, pages_after in journal:
        row = rows.setdefault(rid, [])
        if pages_after == 0:
            for p in row:
                heapq.heappush(free, p)
            final[rid] = list(row)
            del rows[rid]
        else:
            while len(row) < pages_after:
                row.append(heapq.heappop(free))
    return final

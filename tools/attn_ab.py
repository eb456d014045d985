"""A/B of the decode attention kernels on one prefilled state: run one decode
step with logits under the current SW_ATTN_FLAT setting and save them, so two
processes (SW_ATTN_FLAT=0 / 1) can be compared; optionally check rows against
the CPU oracle (emulated bf16 storage points).

  SW_ATTN_FLAT=1 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 64 --prompt 1000 --save /tmp/a.npy
"""
import argparse
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from oracle import model as M
from paper_2505_03763_b200 import runtime


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="LLAMA_1B")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=str, default="1000", help="N or lo..hi (per-row lengths, seeded)")
    ap.add_argument("--save", default="")
    ap.add_argument("--oracle", type=int, default=0)
    args = ap.parse_args()
    d = dataclasses.replace(getattr(M, args.model), n_layers=args.layers)
    B = args.batch
    if ".." in args.prompt:
        lo, hi = map(int, args.prompt.split(".."))
        rng = np.random.default_rng(7)
        lens = [int(x) for x in rng.integers(lo, hi + 1, size=B)]
    else:
        lens = [int(args.prompt)] * B
    pages_per = (max(lens) + 1 + 15) // 16 + 1
    eng = runtime.Engine(d, max_prefill_tokens=max(min(sum(lens), 32768), 64), max_decode_batch=B,
                         n_pages=B * pages_per + 8, n_slots=B, max_pages_per_slot=pages_per, max_out=8)
    # scattered physical pages: row i uses pages i, i + B, i + 2B, ...
    rows = [[i + B * j for j in range(pages_per)] for i in range(B)]
    prompts = [M.prompt_tokens(d.seed, i, lens[i], d.vocab) for i in range(B)]
    i0 = 0
    while i0 < B:
        i1, tot = i0, 0
        while i1 < B and tot + lens[i1] <= 32768:
            tot += lens[i1]
            i1 += 1
        idx = list(range(i0, i1))
        eng.prefill(idx, [prompts[i] for i in idx], [rows[i][:(lens[i] + 15) // 16] for i in idx], logits=False)
        i0 = i1
    toks = [int(p[-1]) for p in prompts]
    newp = [rows[i][lens[i] // 16] if lens[i] % 16 == 0 else -1 for i in range(B)]
    lg = eng.decode(list(range(B)), lens, tokens=toks, new_page=newp, logits=True)
    torch.cuda.synchronize()
    print(f"SW_ATTN_FLAT={os.environ.get('SW_ATTN_FLAT', '1')}: logits[0,:4] {lg[0, :4]}", flush=True)
    if args.save:
        np.save(args.save, lg)
    if args.oracle:
        N = args.oracle
        o = M.OracleModel(d, emulate_bf16=True)
        o.prefill(prompts[:N], [r[:(lens[i] + 15) // 16] for i, r in enumerate(rows[:N])])
        ref = o.decode(toks[:N], lens[:N], [r[:(lens[i] + 16) // 16] for i, r in enumerate(rows[:N])])
        rel = np.linalg.norm(lg[:N] - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(f"oracle (emulated bf16) per-row rel-L2 max {rel.max():.3e} mean {rel.mean():.3e}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

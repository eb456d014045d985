"""Profiling driver: one prefill batch and one decode step of the Llama-1B (or
8B) shape, bracketed by cudaProfilerStart/Stop so ncu
(--profile-from-start off) captures exactly the region of interest.

  python tools/profile_step.py --model LLAMA_1B --batch 64 --prompt 512 --region decode
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from oracle import model as M
from paper_2505_03763_b200 import runtime


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="LLAMA_1B")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--region", choices=["decode", "prefill"], default="decode")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--graphs", type=int, default=1)
    args = ap.parse_args()
    d = getattr(M, args.model)
    B, S = args.batch, args.prompt
    pages_per = (S + 64 + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=max(B * S, 64), max_decode_batch=B, n_pages=B * pages_per + 8,
                         n_slots=B, max_pages_per_slot=pages_per, max_out=64)
    rows = [list(range(i * pages_per, (i + 1) * pages_per)) for i in range(B)]
    prompts = [M.prompt_tokens(d.seed, i, S, d.vocab) for i in range(B)]
    cudart = torch.cuda.cudart()
    if args.region == "prefill":
        eng.prefill(list(range(B)), prompts, [r[:(S + 15) // 16] for r in rows], logits=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStart()
        t = time.perf_counter()
        eng.prefill(list(range(B)), prompts, [r[:(S + 15) // 16] for r in rows], logits=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStop()
        print(f"prefill {B}x{S}: {1e3 * (time.perf_counter() - t):.2f} ms wall")
        return
    eng.prefill(list(range(B)), prompts, [r[:(S + 15) // 16] for r in rows], logits=False)
    pos = [S] * B
    for _ in range(3):  # warm (captures the graph)
        eng.decode(list(range(B)), pos, tokens=None, new_page=[-1] * B, logits=False)
    torch.cuda.synchronize()
    cudart.cudaProfilerStart()
    t = time.perf_counter()
    for _ in range(args.steps):
        eng.decode(list(range(B)), pos, tokens=None, new_page=[-1] * B, logits=False)
    torch.cuda.synchronize()
    cudart.cudaProfilerStop()
    print(f"decode b={B} ctx={S}: {1e3 * (time.perf_counter() - t) / args.steps:.3f} ms/step wall")


if __name__ == "__main__":
    main()

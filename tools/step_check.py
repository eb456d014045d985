"""A/B of the two decode paths on one engine: per-projection kernels
(SW_DECODE_STEP=0) vs the persistent decode-step kernel (SW_DECODE_STEP=1).
Same prefilled KV state, same step inputs: logits rel-L2 and greedy-token
agreement, then device time per step of each path under CUDA-graph replay.

  python tools/step_check.py --model LLAMA_1B --batch 64 --prompt 512
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
    ap.add_argument("--model", default="TINY")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--oracle", type=int, default=0, help="also check the first N rows against the CPU oracle")
    args = ap.parse_args()
    d = getattr(M, args.model)
    if args.layers:
        import dataclasses

        d = dataclasses.replace(d, n_layers=args.layers)
    B, S = args.batch, args.prompt
    pages_per = (S + args.steps + 16 + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=max(B * S, 64), max_decode_batch=max(B, 1), n_pages=B * pages_per + 8,
                         n_slots=B, max_pages_per_slot=pages_per, max_out=args.steps + 8)
    rows = [list(range(i * pages_per, (i + 1) * pages_per)) for i in range(B)]
    prompts = [M.prompt_tokens(d.seed, i, S, d.vocab) for i in range(B)]
    eng.prefill(list(range(B)), prompts, [r[: (S + 15) // 16] for r in rows], logits=False)
    torch.cuda.synchronize()
    modes = [int(x) for x in args.modes.split(",")]
    pos = [S] * B
    toks = [int(p[-1]) for p in prompts]
    res = {}

    def newp(p):  # the page a step at position p starts (its first token), else -1
        return [rows[i][p // 16] if p % 16 == 0 else -1 for i in range(B)]

    for mode in modes:
        os.environ["SW_DECODE_STEP"] = str(mode)
        lg = eng.decode(list(range(B)), pos, tokens=toks, new_page=newp(S), logits=True)
        res[mode] = lg
        print(f"mode {mode}: logits[0,:4] {lg[0, :4]}", flush=True)
    if len(modes) == 2:
        a, b = res[modes[0]], res[modes[1]]
        rel = np.linalg.norm(a - b) / np.linalg.norm(a)
        agree = np.mean(np.argmax(a, 1) == np.argmax(b, 1))
        print(f"logits rel-L2 {rel:.3e}  argmax agreement {agree:.3f}  max|d| {np.abs(a - b).max():.3e}", flush=True)
    if args.oracle:
        N = args.oracle
        for emu in (True, False):
            o = M.OracleModel(d, emulate_bf16=emu)
            o.prefill(prompts[:N], [r[: (S + 15) // 16] for r in rows[:N]])
            ref = o.decode(toks[:N], pos[:N], [r[: (S + 16) // 16] for r in rows[:N]])
            for mode in modes:
                g = res[mode][:N]
                rel = np.linalg.norm(g - ref, axis=1) / np.linalg.norm(ref, axis=1)
                print(f"oracle emulate_bf16={emu}: mode {mode} per-row rel-L2 max {rel.max():.3e} mean {rel.mean():.3e}",
                      flush=True)
            del o
    # timing: graph replay, the step's own last tokens fed back (tokens=None)
    for mode in modes:
        os.environ["SW_DECODE_STEP"] = str(mode)
        for i in range(3):
            eng.decode(list(range(B)), [S + 1 + i] * B, tokens=None, new_page=newp(S + 1 + i), logits=False)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        for i in range(args.steps):
            eng.decode(list(range(B)), [S + 4 + i] * B, tokens=None, new_page=newp(S + 4 + i), logits=False)
        e1.record(st)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        print(f"mode {mode}: {e0.elapsed_time(e1) / args.steps:.3f} ms/step device, {1e3 * wall:.3f} ms/step wall",
              flush=True)
    eng.close()


if __name__ == "__main__":
    main()

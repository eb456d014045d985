"""Device time of one decode step: K steps enqueued back to back through the
C-ABI (sw_decode_enqueue, CUDA-graph path) on one stream, bracketed by CUDA
events -- no host synchronisation between steps.

  python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 [--steps 50]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from oracle import model as M
import paper_2505_03763_b200 as sw
from paper_2505_03763_b200 import runtime


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="LLAMA_1B")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    d = getattr(M, args.model)
    B, S = args.batch, args.prompt
    pages_per = (S + 64 + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=max(min(B * S, 32768), 64), max_decode_batch=B,
                         n_pages=B * pages_per + 8, n_slots=B, max_pages_per_slot=pages_per, max_out=64)
    rows = [list(range(i * pages_per, (i + 1) * pages_per)) for i in range(B)]
    prompts = [M.prompt_tokens(d.seed, i, S, d.vocab) for i in range(B)]
    chunk = max(1, 32768 // S)
    for c0 in range(0, B, chunk):
        idx = list(range(c0, min(B, c0 + chunk)))
        eng.prefill(idx, [prompts[i] for i in idx], [rows[i][:(S + 15) // 16] for i in idx], logits=False)
    st = torch.cuda.Stream()
    slots = (ctypes.c_int32 * B)(*range(B))
    pos = (ctypes.c_int32 * B)(*([S] * B))
    newp = (ctypes.c_int32 * B)(*([-1] * B))
    b = sw.Batch(n=B, slots=slots, positions=pos)
    b.new_page = newp
    L = sw.lib()
    sp = ctypes.c_void_p(st.cuda_stream)

    def step():
        sw.check(L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(b), sp))

    with torch.cuda.stream(st):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        best = None
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.steps):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            best = ms if best is None else min(best, ms)
    print(f"{args.model} b={B} ctx={S}: {best:.4f} ms/step device (best of {args.reps} x {args.steps})", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

"""Device time of a multi-prompt prefill launch (sw_prefill_enqueue, back to back on one stream, CUDA
events): n prompts x L tokens of the given model, logits off.

  python tools/prefill_time.py --model LLAMA_8B --prompts 8 --len 1088 [--reps 5]
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
    ap.add_argument("--model", default="LLAMA_8B")
    ap.add_argument("--prompts", type=int, default=8)
    ap.add_argument("--len", type=int, default=1088)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    d = getattr(M, a.model)
    n, L = a.prompts, a.len
    per = (L + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=max(n * L, 256), max_decode_batch=8, n_pages=n * per + 8, n_slots=n,
                         max_pages_per_slot=per, max_out=8)
    keep = []

    def arr(xs):
        x = (ctypes.c_int32 * len(xs))(*[int(v) for v in xs])
        keep.append(x)
        return x

    toks = []
    for i in range(n):
        toks += [int(t) for t in M.prompt_tokens(d.seed, i, L, d.vocab)]
    b = sw.Batch(n=n, slots=arr(range(n)), n_tokens=arr([L] * n), tokens=arr(toks),
                 page_rows=arr([i * per + j for i in range(n) for j in range(per)]), out_index=arr([0] * n))
    st = torch.cuda.Stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    lib = sw.lib()
    with torch.cuda.stream(st):
        for _ in range(2):
            sw.check(lib.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(b), sp))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            sw.check(lib.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(b), sp))
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{a.model} prefill {n} x {L}: {ms:.2f} ms, {n * L / ms * 1e3:.0f} tok/s", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

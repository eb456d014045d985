"""Cost of a fused mixed step against its parts, on the device (CUDA events, one
stream, launches back to back): a decode step of B rows at context S, a prefill
of C prompt tokens, and one sw_mixed_enqueue launch carrying both.

  python tools/fused_step.py --model LLAMA_8B --batch 256 --ctx 1216 --chunks 512,1024,2048,4096,8192
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
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=1216)
    ap.add_argument("--chunks", default="512,1024,2048,4096,8192")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--once", type=int, default=0, help="ncu: one decode, one prefill, one fused launch of this chunk")
    args = ap.parse_args()
    d = getattr(M, args.model)
    B, S = args.batch, args.ctx
    chunks = [int(c) for c in args.chunks.split(",")] if args.chunks != "none" else [128]
    cmax = max(chunks)
    per_d = (S + 16 + 15) // 16  # decode rows' pages
    per = max(per_d, (cmax + 15) // 16)
    n_slots = B + 1
    eng = runtime.Engine(d, max_prefill_tokens=32768, max_decode_batch=B, n_pages=B * per_d + per + 8,
                         n_slots=n_slots, max_pages_per_slot=per, max_out=16)
    rows = [list(range(i * per_d, (i + 1) * per_d)) for i in range(B)] + [list(range(B * per_d, B * per_d + per))]
    prompts = [M.prompt_tokens(d.seed, i, S, d.vocab) for i in range(B)]
    step = max(1, 32768 // S)
    for c0 in range(0, B, step):
        idx = list(range(c0, min(B, c0 + step)))
        eng.prefill(idx, [prompts[i] for i in idx], [rows[i][:(S + 15) // 16] for i in idx], logits=False)
    L = sw.lib()
    st = torch.cuda.Stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    keep = []

    def arr(xs):
        a = (ctypes.c_int32 * len(xs))(*xs)
        keep.append(a)
        return a

    db = sw.Batch(n=B, slots=arr(list(range(B))), positions=arr([S] * B))
    db.new_page = arr([-1] * B)

    def pre_batch(C):
        p = M.prompt_tokens(d.seed, 10_000 + C, C, d.vocab)
        b = sw.Batch(n=1, slots=arr([B]), n_tokens=arr([C]), tokens=arr([int(x) for x in p]),
                     page_rows=arr(rows[B][:(C + 15) // 16]), out_index=arr([0]))
        return b

    def timed(fn, n):
        with torch.cuda.stream(st):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            best = 1e30
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(n):
                    fn()
                e1.record(st)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / n)
        return best

    if args.once:
        pb = pre_batch(args.once)
        with torch.cuda.stream(st):
            for f in (lambda: L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(db), sp),
                      lambda: L.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(pb), sp),
                      lambda: L.sw_mixed_enqueue(eng.model, eng.kv, ctypes.byref(pb), ctypes.byref(db), sp)):
                torch.cuda.synchronize()
                sw.check(f())
                torch.cuda.synchronize()
        eng.close()
        return
    t_dec = timed(lambda: sw.check(L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(db), sp)), 10)
    print(f"{args.model} decode step b={B} ctx={S}: {t_dec:.3f} ms", flush=True)
    # the same token step through the prefill kernels (normal-mode CTA-pair GEMMs, T = B rows)
    eb = sw.Batch(n=0, slots=arr([0]), n_tokens=arr([0]), tokens=arr([0]), page_rows=arr([0]), out_index=arr([0]))
    t_dp = timed(lambda: sw.check(L.sw_mixed_enqueue(eng.model, eng.kv, ctypes.byref(eb), ctypes.byref(db), sp)), 10)
    print(f"{args.model} decode step b={B} ctx={S} through the prefill kernels: {t_dp:.3f} ms", flush=True)
    if args.chunks == "none":
        eng.close()
        return
    for C in chunks:
        pb = pre_batch(C)
        t_pre = timed(lambda: sw.check(L.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(pb), sp)), 3)
        t_mix = timed(lambda: sw.check(L.sw_mixed_enqueue(eng.model, eng.kv, ctypes.byref(pb), ctypes.byref(db), sp)), 3)
        print(f"  chunk {C:5d}: prefill {t_pre:8.3f} ms  decode+prefill {t_dec + t_pre:8.3f} ms  fused {t_mix:8.3f} ms"
              f"  fused/sum {t_mix / (t_dec + t_pre):.3f}  prefill tok/s alone {C / t_pre * 1e3:9.0f}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

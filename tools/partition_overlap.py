"""Kernel-level phase concurrency on green-context SM partitions.

For each decode partition size D: a decode step stream (b rows at context S,
CUDA-graph path) on D SMs and a prefill (P prompts x Sp tokens) on the other
148-D SMs, first each alone on its partition, then both at once.  Reports
  eff = t_prefill(whole GPU)/t_prefill(shared) + t_step(whole GPU)/t_step(shared)
(1.0 = time slicing, 2.0 = both phases at whole-GPU speed) -- the number the
split-phase engine's gain is bounded by.  All times are CUDA events on the
launching streams.

  python tools/partition_overlap.py --model LLAMA_8B --batch 64 --ctx 1024 --prompts 8 --prompt-len 1024 \
      --decode-sms 32,48,64,80
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2505_03763_b200 as sw
from paper_2505_03763_b200 import runtime, shapes
from oracle import model as M


def i32(xs):
    return (ctypes.c_int32 * len(xs))(*[int(x) for x in xs])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="LLAMA_8B")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--prompts", type=int, default=8)
    ap.add_argument("--prompt-len", type=int, default=1024)
    ap.add_argument("--decode-sms", default="32,48,64,80")
    ap.add_argument("--stream-gb", type=float, default=0.0, help="replace decode steps by a read stream of this size")
    args = ap.parse_args()
    d = getattr(shapes, args.model)
    B, S, P, Sp = args.batch, args.ctx, args.prompts, args.prompt_len
    pages_dec = (S + 64 + 15) // 16
    pages_pre = (Sp + 15) // 16
    n_pages = B * pages_dec + P * pages_pre + 8
    eng = runtime.Engine(d, max_prefill_tokens=min(32768, max(P * Sp, 64)), max_decode_batch=B, n_pages=n_pages,
                         n_slots=B + P, max_pages_per_slot=max(pages_dec, pages_pre), max_out=64)
    L = sw.lib()
    rows = [list(range(i * pages_dec, (i + 1) * pages_dec)) for i in range(B)]
    chunk = max(1, 32768 // S)
    for c0 in range(0, B, chunk):
        idx = list(range(c0, min(B, c0 + chunk)))
        eng.prefill(idx, [M.prompt_tokens(d.seed, i, S, d.vocab) for i in idx],
                    [rows[i][:(S + 15) // 16] for i in idx], logits=False)
    # decode batch: one token at position S for every row (re-run each step: same bytes, same work)
    dkeep = [i32(range(B)), i32([S] * B), i32([-1] * B)]
    db = sw.Batch(n=B, slots=dkeep[0], positions=dkeep[1])
    db.new_page = dkeep[2]
    # prefill batch: P prompts of Sp tokens into slots B..B+P-1 (their own pages)
    base = B * pages_dec
    ptoks = np.concatenate([M.prompt_tokens(d.seed, 1000 + i, Sp, d.vocab) for i in range(P)])
    pkeep = [i32(range(B, B + P)), i32([Sp] * P), i32(ptoks),
             i32([base + i * pages_pre + j for i in range(P) for j in range(pages_pre)]), i32([0] * P)]
    pb = sw.Batch(n=P, slots=pkeep[0], n_tokens=pkeep[1], tokens=pkeep[2], page_rows=pkeep[3], out_index=pkeep[4])

    # --stream: the decode phase replaced by a pure HBM read stream of the same bytes as one step
    # (torch reduction over a buffer > L2), to separate interference in the memory system from the
    # decode kernels' own partition behaviour
    sbuf = torch.empty(int(args.stream_gb * (1 << 30)) // 4, dtype=torch.float32, device="cuda") if args.stream_gb else None
    sink = torch.empty(1, dtype=torch.float32, device="cuda")

    def dec(st):
        if sbuf is not None:
            with torch.cuda.stream(torch.cuda.ExternalStream(st)):
                torch.sum(sbuf, dim=0, out=sink[0])
            return
        sw.check(L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(db), ctypes.c_void_p(st)))

    def pre(st):
        sw.check(L.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(pb), ctypes.c_void_p(st)))

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def time_alone(fn, st, k):
        s = torch.cuda.ExternalStream(st)
        for _ in range(2):
            fn(st)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(s)
        for _ in range(k):
            fn(st)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    full = torch.cuda.Stream()
    t_dec_full = time_alone(dec, full.cuda_stream, 30)
    t_pre_full = time_alone(pre, full.cuda_stream, 3)
    flops = 2.0 * P * Sp * (d.n_layers * (d.d_model * (d.n_heads + 2 * d.n_kv_heads) * d.head_dim +
                                          d.n_heads * d.head_dim * d.d_model + 3 * d.d_model * d.ffn_dim))
    print(f"{args.model} decode b={B} ctx={S}: whole GPU {t_dec_full:.3f} ms/step | prefill {P}x{Sp}: "
          f"{t_pre_full:.2f} ms ({flops / t_pre_full / 1e9:.0f} TFLOP/s matmul)", flush=True)
    for ds in [int(x) for x in args.decode_sms.split(",")]:
        dp, pp, dn, pn = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int(), ctypes.c_int()
        sw.check(L.sw_sm_partition(0, ds, ctypes.byref(dp), ctypes.byref(pp), ctypes.byref(dn), ctypes.byref(pn)))
        t_dec = time_alone(dec, dp.value, 30)
        t_pre = time_alone(pre, pp.value, 3)
        # both at once: decode steps keep running for the prefill's duration
        k = max(3, int(round(t_pre / t_dec)))
        sd, sp_ = torch.cuda.ExternalStream(dp.value), torch.cuda.ExternalStream(pp.value)
        torch.cuda.synchronize()
        go = ev()
        go.record(torch.cuda.current_stream())
        sd.wait_event(go)
        sp_.wait_event(go)
        p0, p1, d0, d1 = ev(), ev(), ev(), ev()
        p0.record(sp_)
        pre(pp.value)
        p1.record(sp_)
        d0.record(sd)
        for _ in range(k):
            dec(dp.value)
        d1.record(sd)
        torch.cuda.synchronize()
        t_pre_sh = p0.elapsed_time(p1)
        t_dec_sh = d0.elapsed_time(d1) / k
        eff = t_pre_full / t_pre_sh + t_dec_full / t_dec_sh
        print(f"decode {dn.value:3d} SMs | prefill {pn.value:3d} SMs : alone step {t_dec:.3f} ms ({t_dec_full / t_dec:.2f}x), "
              f"prefill {t_pre:.2f} ms ({t_pre_full / t_pre:.2f}x) | shared step {t_dec_sh:.3f} ms, prefill {t_pre_sh:.2f} ms "
              f"(window {k} steps) | eff {eff:.2f}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

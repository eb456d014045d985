"""Is the decode attention clock-sensitive?  The bench times the dominant
kernel (paged-KV decode attention, 8B, 256 rows x ctx 1217) after the engine
runs, while the board may still be power-managing.  This times the same probe
(bench.roofline_decode_attention) on a cool GPU, right after a prefill heat
soak (the prefill GEMM holds the board at its power cap), and after idling,
with the SM clock sampled during each measurement.

  python tools/attn_clock_probe.py [--soak 8]
"""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
import paper_2505_03763_b200 as sw
from paper_2505_03763_b200 import runtime, shapes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--soak", type=float, default=8.0)
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=1216)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    desc = shapes.LLAMA_8B
    peaks, _ = bench.load_peaks()
    per = (args.ctx + 1 + 15) // 16
    eng = runtime.Engine(desc, max_prefill_tokens=32768, max_decode_batch=args.rows, n_pages=args.rows * per + 64,
                         n_slots=args.rows + 8, max_pages_per_slot=per + 1, max_out=8)
    d, F = desc.d_model, desc.ffn_dim
    x = torch.randn(8192, d, device="cuda").bfloat16()
    y = torch.empty(8192, F, device="cuda", dtype=torch.bfloat16)
    w0 = eng.tensor("layer0.wgu")[0]

    def soak(sec):
        t0 = time.time()
        while time.time() - t0 < sec:
            for _ in range(20):
                sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w0),
                                             ctypes.c_void_p(y.data_ptr()), 8192, 2 * F, d, 2,
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
            torch.cuda.synchronize()

    state = {"prefilled": False}

    big = torch.empty(2 << 30, device="cuda", dtype=torch.bfloat16)  # 4 GiB: a read-only stream (sum) and a copy
    big.fill_(1.0)
    dst = torch.empty(1 << 30, device="cuda", dtype=torch.bfloat16)

    def streams():
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        for _ in range(5):
            big.sum(dtype=torch.float32)
        e1.record()
        for _ in range(5):
            dst.copy_(big[: 1 << 30])
        e2.record()
        torch.cuda.synchronize()
        rd = 5 * big.numel() * 2 / (e0.elapsed_time(e1) / 1e3) / 1e9
        cp = 5 * 2 * dst.numel() * 2 / (e1.elapsed_time(e2) / 1e3) / 1e9
        return rd, cp

    def probe(tag, settle=0.0):
        with bench.ClockSampler(0) as c:
            r = bench.roofline_decode_attention(eng, desc, args.rows, args.ctx, peaks, reps=args.reps,
                                                prefilled=state["prefilled"], settle_s=settle)
        state["prefilled"] = True
        s = c.summary()
        rd, cp = streams()  # right after, in the same power state
        print(f"{tag:28s} {r['us_per_launch']:7.2f} us/layer  {r['achieved']:7.1f} GB/s  frac {r['frac']:.4f}  "
              f"SM {s['sm_mhz']} MHz  {s['reasons']} | torch read stream {rd:7.1f} GB/s, copy {cp:7.1f} GB/s",
              flush=True)

    probe("right after its prefill")
    probe("again (no settle)")
    probe("after 5 s settle", settle=5.0)
    soak(args.soak)
    probe(f"after {args.soak:.0f} s prefill soak")
    time.sleep(5)
    probe("after 5 s idle")
    # concurrent with the soak: the power state of a real split run
    soak(args.soak)
    probe("after second soak")
    eng.close()


if __name__ == "__main__":
    main()

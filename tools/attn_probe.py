"""Decode attention alone (sw_op_decode_attention, every layer) at R rows x ctx, 8B shape: achieved
HBM bandwidth of the kernel the step picks (SW_ATTN_FLAT=0/1/2 to force per-unit / flat / auto).

  python tools/attn_probe.py --rows 256 --ctx 1216
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2505_03763_b200 import runtime, shapes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=1216)
    ap.add_argument("--model", default="LLAMA_8B")
    a = ap.parse_args()
    d = getattr(shapes, a.model)
    per = (a.ctx + 1 + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=32768, max_decode_batch=a.rows, n_pages=a.rows * per + 8,
                         n_slots=a.rows, max_pages_per_slot=per, max_out=8)
    peaks, _ = bench.load_peaks()
    r = bench.roofline_decode_attention(eng, d, a.rows, a.ctx, peaks)
    print(f"{a.model} rows={a.rows} ctx={a.ctx} SW_ATTN_FLAT={os.environ.get('SW_ATTN_FLAT', '2')}: "
          f"{r['us_per_launch']} us/layer, {r['achieved']} GB/s, frac {r['frac']}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()

"""Decode-shape projections at b rows: this repo's decode GEMM (sw_op_gemm,
swap-AB tcgen05 + fused epilogue) vs cuBLAS (torch.matmul, no epilogue), both
replayed from a CUDA graph over 8 weight copies (> L2), CUDA events.

  python tools/dec_vs_cublas.py [rows ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03763_b200 as sw

SHAPES = [("8b.qkv", 6144, 4096, 4), ("8b.wo", 4096, 4096, 1), ("8b.gu", 28672, 4096, 2), ("8b.wd", 4096, 14336, 1),
          ("1b.qkv", 3072, 2048, 4), ("1b.wo", 2048, 2048, 1), ("1b.gu", 16384, 2048, 2), ("1b.wd", 2048, 8192, 1)]
COPIES, REPS = 8, 24


def graph_us(go):
    st = torch.cuda.current_stream()
    for i in range(COPIES):
        go(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(REPS):
            go(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / REPS)
    return best


def main():
    rows_list = [int(a) for a in sys.argv[1:]] or [64, 128, 256]
    for rows in rows_list:
        for name, feat, K, epi in SHAPES:
            Ws = [torch.randn(feat, K, device="cuda").bfloat16() for _ in range(COPIES)]
            X = torch.randn(rows, K, device="cuda").bfloat16()
            out = torch.zeros(rows, feat, device="cuda")
            Y = torch.empty(rows, feat, device="cuda", dtype=torch.bfloat16)

            def ours(i):
                sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Ws[i % COPIES].data_ptr()),
                                             ctypes.c_void_p(out.data_ptr()), rows, feat, K, epi,
                                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

            def cublas(i):
                torch.matmul(X, Ws[i % COPIES].t(), out=Y)

            a, b = graph_us(ours), graph_us(cublas)
            gb = feat * K * 2 / 1e3
            print(f"b={rows:3d} {name:7s} F={feat:5d} K={K:5d}: ours {a:7.2f} us {gb / a:6.0f} GB/s | "
                  f"cuBLAS {b:7.2f} us {gb / b:6.0f} GB/s | ours/cuBLAS time {a / b:5.2f}", flush=True)
            del Ws


if __name__ == "__main__":
    main()

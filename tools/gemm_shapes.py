"""Decode-shape GEMM timing under CUDA-graph replay (no host launch cost):
the Llama projections at b rows with their real epilogues."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03763_b200 as sw

SHAPES = [("1b.qkv", 3072, 2048, 4), ("1b.wo", 2048, 2048, 1), ("1b.gu", 16384, 2048, 2), ("1b.wd", 2048, 8192, 1),
          ("1b.lm", 128256, 2048, 4), ("8b.qkv", 6144, 4096, 4), ("8b.wo", 4096, 4096, 1), ("8b.gu", 28672, 4096, 2),
          ("8b.wd", 4096, 14336, 1)]


def t(feat, K, epi, rows, reps=int(os.environ.get("REPS", "20")), copies=int(os.environ.get("COPIES", "4"))):
    Ws = [torch.randn(feat, K, device="cuda").bfloat16() for _ in range(copies)]
    X = torch.randn(rows, K, device="cuda").bfloat16()
    out = torch.zeros(rows, feat, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sp = ctypes.c_void_p(st.cuda_stream)

        def go(i):
            sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Ws[i % copies].data_ptr()),
                                         ctypes.c_void_p(out.data_ptr()), rows, feat, K, epi, sp))

        for i in range(copies):
            go(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(reps):
                go(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    return us, feat * K * 2 / us / 1e3


if __name__ == "__main__":
    rows = int(os.environ.get("ROWS", "64"))
    only = os.environ.get("ONLY")
    for name, feat, K, epi in SHAPES:
        if only and name not in only.split(","):
            continue
        us, gbs = t(feat, K, epi, rows)
        print(f"{name:8s} b={rows}: {us:8.2f} us {gbs:8.1f} GB/s", flush=True)

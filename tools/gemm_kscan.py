"""Fixed-cost vs per-K-block cost of the swap-AB decode GEMM: time one tile
(128 weight rows) and 148 tiles (one CTA per SM) for growing K, via a CUDA
graph of 20 launches (no host launch overhead in the measurement)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03763_b200 as sw


def t(feat, K, rows=64, epi=4, reps=20):
    copies = 4
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
    pass
    for feat in (128, 128 * 148):
        for K in (64, 256, 1024, 2048, 4096, 8192):
            us, gbs = t(feat, K)
            print(f"tiles={feat // 128:4d} K={K:5d}: {us:8.2f} us  {gbs:8.1f} GB/s", flush=True)

"""Decode GEMM tuning sweep: time the swap-AB tcgen05 GEMM on the Llama
projection shapes for several split-K factors / smem budgets (env overrides
read by the library at first use, so each config runs in a fresh process)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03763_b200 as sw

SHAPES = {  # name: (features, K, epilogue)
    "1b.qkv": (3072, 2048, 4), "1b.wo": (2048, 2048, 1), "1b.gu": (16384, 2048, 2), "1b.wd": (2048, 8192, 1),
    "1b.lm": (128256, 2048, 3),
    "8b.qkv": (6144, 4096, 4), "8b.wo": (4096, 4096, 1), "8b.gu": (28672, 4096, 2), "8b.wd": (4096, 14336, 1),
}


def time_shape(feat, K, epi, rows, reps=30, copies=8):
    Ws = [torch.randn(feat, K, device="cuda").bfloat16() for _ in range(copies)]  # rotate > L2
    X = torch.randn(rows, K, device="cuda").bfloat16()
    out = torch.zeros(rows, feat, device="cuda", dtype=torch.float32)
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)

    def go(i):
        if epi == 3:
            return  # argmax needs keys; use STORE_F32 timing instead
        sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Ws[i % copies].data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()), rows, feat, K, epi, sp))

    if epi == 3:
        epi = 4
    for i in range(copies):
        go(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(reps):
        go(i)
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    gbs = feat * K * 2 / (us * 1e-6) / 1e9
    return us, gbs


if __name__ == "__main__":
    rows = int(os.environ.get("ROWS", "64"))
    res = {}
    for name, (feat, K, epi) in SHAPES.items():
        if epi == 2:
            pass
        us, gbs = time_shape(feat, K, epi if epi != 4 else 4, rows)
        res[name] = (round(us, 2), round(gbs, 1))
    print(json.dumps({"rows": rows, "splits": os.environ.get("SW_GEMM_SPLITS", "auto"),
                      "small": os.environ.get("SW_GEMM_SMALL", "auto"), "res": res}))

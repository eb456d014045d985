"""The prefill projection GEMMs (tcgen05 CTA-pair kernel through sw_op_gemm,
store epilogue) against cuBLAS (torch.matmul, bf16) on the same shapes,
timed back to back with CUDA events over a graph of 20 launches, with the SM
clock sampled -- is there throughput left on the table at the power cap?

  python tools/gemm_vs_cublas.py [--tokens 4096,8192]
"""
import argparse
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2505_03763_b200 as sw


def timed(fn, reps=20):
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps / 1e3
        best = t if best is None else min(best, t)
    return best


def sm_mhz():
    out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="4096,8192")
    args = ap.parse_args()
    L = sw.lib()
    shapes = [("8B qkv", 6144, 4096), ("8B wo", 4096, 4096), ("8B gate/up", 28672, 4096), ("8B down", 4096, 14336),
              ("1B gate/up", 16384, 2048)]
    for T in [int(x) for x in args.tokens.split(",")]:
        for name, N, K in shapes:
            a = torch.randn(T, K, device="cuda").bfloat16()
            w = torch.randn(N, K, device="cuda").bfloat16() * 0.02
            c = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)

            def ours():
                sw.check(L.sw_op_gemm(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                      ctypes.c_void_p(c.data_ptr()), T, N, K, 0,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

            def cublas():
                torch.matmul(a, w.t(), out=c)

            fl = 2.0 * T * N * K
            ours()  # first call configures the kernel and allocates the op workspace (outside capture)
            cublas()
            t_o = timed(ours)
            mo = sm_mhz()
            t_c = timed(cublas)
            mc = sm_mhz()
            print(f"T={T:5d} {name:<11s} N={N:5d} K={K:5d}: ours {fl / t_o / 1e12:7.1f} TFLOP/s ({mo} MHz)  "
                  f"cuBLAS {fl / t_c / 1e12:7.1f} TFLOP/s ({mc} MHz)  ours/cuBLAS {t_c / t_o:.3f}", flush=True)


if __name__ == "__main__":
    main()

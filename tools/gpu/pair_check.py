"""Numerics of the prefill GEMM (sw_op_gemm, normal mode) vs torch, for the CTA-pair
and single-CTA variants (SW_GEMM_PAIR read once per process: run twice)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2505_03763_b200 as sw
L = sw.lib()
torch.manual_seed(0)
for (M, N, K) in [(512, 512, 256), (4096, 2048, 2048), (16384, 16384, 2048), (1000, 3072, 2048), (300, 768, 256)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream()
    sw.check(L.sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                          M, N, K, 0, ctypes.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    ref = (x.float() @ w.float().t())
    rel = ((y.float() - ref).norm() / ref.norm()).item()
    # timing
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        L.sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                     M, N, K, 0, ctypes.c_void_p(st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    print(f"PAIR={os.environ.get('SW_GEMM_PAIR','1')} M={M} N={N} K={K}: rel {rel:.2e}  {us:.1f} us  {2*M*N*K/us/1e6:.1f} TFLOP/s", flush=True)

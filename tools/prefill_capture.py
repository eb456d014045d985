"""ncu target for the prefill projections at the 8B shape: gate/up (SwiGLU), Wo and
Wd (residual-add epilogue) at T tokens, two rounds over distinct layers' weights.

  ncu --set full --clock-control none -k regex:gemm_tc --launch-skip 3 -c 3 \
      -o gpurun_out/pre python tools/prefill_capture.py --tokens 4096
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2505_03763_b200 as sw
from oracle import model as M
from paper_2505_03763_b200 import runtime


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    a = ap.parse_args()
    d = M.LLAMA_8B
    T = a.tokens
    eng = runtime.Engine(d, max_prefill_tokens=256, max_decode_batch=8, n_pages=64, n_slots=8, max_pages_per_slot=8,
                         max_out=8)
    x = torch.randn(T, d.ffn_dim, device="cuda").bfloat16()
    act = torch.empty(T, d.ffn_dim, device="cuda", dtype=torch.bfloat16)
    res = torch.randn(T, d.d_model, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L = sw.lib()
    xp = ctypes.c_void_p(x.data_ptr())
    for r in range(2):
        l = 2 * r
        L.sw_op_gemm(xp, ctypes.c_void_p(eng.tensor(f"layer{l}.wgu")[0]), ctypes.c_void_p(act.data_ptr()), T,
                     2 * d.ffn_dim, d.d_model, 2, st)
        L.sw_op_gemm(xp, ctypes.c_void_p(eng.tensor(f"layer{l}.wo")[0]), ctypes.c_void_p(res.data_ptr()), T,
                     d.d_model, d.n_heads * d.head_dim, 1, st)
        L.sw_op_gemm(xp, ctypes.c_void_p(eng.tensor(f"layer{l}.wd")[0]), ctypes.c_void_p(res.data_ptr()), T,
                     d.d_model, d.ffn_dim, 1, st)
    torch.cuda.synchronize()
    print("ok")
    eng.close()


if __name__ == "__main__":
    main()

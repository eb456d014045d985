"""Phase timeline of one stream-K decode GEMM launch (SW_DSK_TRACE=1 globaltimer
stamps per CTA): start, first k-block ready, last MMA issued, main loop joined,
reduction waits/ends, exit -- us after the earliest CTA start.

  SW_DSK_TRACE=1 python tools/dsk_trace.py F K epi rows
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2505_03763_b200 as sw


def main():
    F, K, epi, rows = (int(a) for a in sys.argv[1:5])
    W = [torch.randn(F, K, device="cuda").bfloat16() for _ in range(4)]
    X = torch.randn(rows, K, device="cuda").bfloat16()
    out = torch.zeros(rows, F, device="cuda")
    lib = sw.lib()
    for i in range(6):
        sw.check(lib.sw_op_gemm(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(W[i % 4].data_ptr()),
                                ctypes.c_void_p(out.data_ptr()), rows, F, K, epi, None))
    torch.cuda.synchronize()
    if os.environ.get("SW_DEC_TRACE"):  # the cluster split-K kernel (gemm_decode.cu)
        buf = (ctypes.c_ulonglong * (512 * 4))()
        lib.sw_dbg_dec_trace(buf, 512 * 4)
        a = np.array(buf, dtype=np.float64).reshape(512, 4)
        names = ["start", "mma_done", "joined", "exit"]
    else:
        buf = (ctypes.c_ulonglong * (256 * 8))()
        lib.sw_dbg_dsk_trace(buf, 256 * 8)
        a = np.array(buf, dtype=np.float64).reshape(256, 8)
        names = ["start", "first_kb", "mma_done", "joined", "wait1", "red1", "wait2", "red2/exit"]
    live = a[:, 0] > 0
    a = a[live]
    t0 = a[:, 0].min()
    print(f"F={F} K={K} epi={epi} rows={rows}: {live.sum()} CTAs")
    for j, n in enumerate(names):
        v = a[:, j]
        v = v[v > 0]
        if len(v) == 0:
            continue
        v = (v - t0) / 1e3
        print(f"  {n:10s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")
        if n == "start":  # CTA start histogram: a second wave shows as a late group
            h, e = np.histogram(v, bins=8)
            print("    start histogram:", " ".join(f"{c}@{x:.1f}" for c, x in zip(h, e[:-1])))


if __name__ == "__main__":
    main()

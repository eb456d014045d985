"""ncu target for bench.py's roofline kernel: the decode gate/up projection
(swap-AB tcgen05 GEMM + SwiGLU, sw_op_gemm mode 2) at the bench's decode batch,
rotating over every layer's weights exactly like bench.roofline_decode_gemm.

  ncu --set full --clock-control none -k regex:gemm_tc --launch-skip 4 -c 2 \
      -o gpurun_out/roof python tools/roofline_capture.py --workload 1b
  python tools/roofline_capture.py --parse gpurun_out/roof.ncu-rep --workload 1b

--parse reads the capture's dram__bytes_{read,write}.sum per launch and merges
them into profiles/roofline_traffic.json, which bench.py reports as
roofline.traffic."""
import argparse
import ctypes
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def capture(workload):
    import torch
    import bench
    import paper_2505_03763_b200 as sw
    from oracle import model as M
    from paper_2505_03763_b200 import runtime

    w = bench.WORKLOADS[workload]
    desc = getattr(M, w["model"])
    eng = runtime.Engine(desc, max_prefill_tokens=256, max_decode_batch=w["max_decode"], n_pages=64, n_slots=8,
                         max_pages_per_slot=8, max_out=8)
    rows, d, F, L = w["max_decode"], desc.d_model, desc.ffn_dim, desc.n_layers
    x = torch.randn(rows, d, device="cuda").bfloat16()
    y = torch.empty(rows, F, device="cuda", dtype=torch.bfloat16)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i in range(L + 4):
        w_ptr = eng.tensor(f"layer{i % L}.wgu")[0]
        sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w_ptr),
                                     ctypes.c_void_p(y.data_ptr()), rows, 2 * F, d, 2, st))
    torch.cuda.synchronize()
    print(f"{L + 4} gate/up launches rows={rows} d={d} F={F}")
    eng.close()


def parse(rep, workload):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}

    def col(r, name):
        i = hdr.index(name)
        return float(r[i].replace(",", "")) * scale[units[i]]

    recs = [dict(kernel=r[hdr.index("Kernel Name")], read=col(r, "dram__bytes_read.sum"),
                 write=col(r, "dram__bytes_write.sum"), t=col(r, "gpu__time_duration.sum")) for r in data]
    n = len(recs)
    traffic = sum(r["read"] + r["write"] for r in recs) / n
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    doc[workload] = {"decode_gate_up_bytes": round(traffic), "launches": n,
                     "dram_read_bytes": round(sum(r["read"] for r in recs) / n),
                     "dram_write_bytes": round(sum(r["write"] for r in recs) / n),
                     "ncu_us_per_launch": round(1e6 * sum(r["t"] for r in recs) / n, 2),
                     "kernel": recs[0]["kernel"], "source": os.path.basename(rep)}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc[workload]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="1b")
    ap.add_argument("--parse", default=None)
    a = ap.parse_args()
    parse(a.parse, a.workload) if a.parse else capture(a.workload)

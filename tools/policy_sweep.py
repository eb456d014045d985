"""Split-vs-serial policy sweep on one engine: tokens/s, p50 TTFT/TBT per spec."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import model as M
from paper_2505_03763_b200 import runtime

model = os.environ.get("MODEL", "LLAMA_1B")
base = os.environ.get("BASE", "n=64;input=512;output=128;seed=1;arrival=zero")
d = getattr(M, model)
n = int(base.split("n=")[1].split(";")[0])
inp = base.split("input=")[1].split(";")[0]
in_max = int(inp.split("..")[-1])
out = int(base.split("output=")[1].split(";")[0])
pages = (in_max + out + 15) // 16
eng = runtime.Engine(d, max_prefill_tokens=32768, max_decode_batch=128, n_pages=n * pages + 64, n_slots=n + 8,
                     max_pages_per_slot=pages + 1, max_out=out + 1)
specs = [s for s in sys.argv[1:]]
for spec in specs:
    full = f"{base};kv_capacity_blocks={n * pages + 64};{spec}"
    eng.run(full)  # warm (graphs, attributes)
    best = None
    for _ in range(2):
        r = eng.run(full)
        tps = r.report["tokens_per_s"]
        best = r if best is None or tps > best.report["tokens_per_s"] else best
    rep = best.report
    print(f"{rep['tokens_per_s']:10.1f} tok/s  p50 ttft {1e3 * rep['p50_ttft_s']:8.2f} ms  p50 tbt {1e3 * rep['p50_tbt_s']:7.3f} ms"
          f"  makespan {rep['makespan_s']:.3f}s  | {spec}", flush=True)
eng.close()

"""configs[2] sweep: 8B shape, n requests, prompts U[128,2048], 256 generated,
Poisson rate swept; serial (continuous batching on one stream) vs split specs.
Usage: RATES=16,64,inf N=512 python tools/cfg3_sweep.py 'spec1' 'spec2' ..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_03763_b200 import runtime, shapes

model = os.environ.get("MODEL", "LLAMA_8B")
n = int(os.environ.get("N", "512"))
inp = os.environ.get("INPUT", "128..2048")
out = int(os.environ.get("OUTPUT", "256"))
rates = os.environ.get("RATES", "32,64,inf").split(",")
reps = int(os.environ.get("REPS", "1"))
max_dec = int(os.environ.get("MAXDEC", "256"))
d = getattr(shapes, model)
in_max = int(inp.split("..")[-1])
pages = (in_max + out + 15) // 16
t0 = time.time()
eng = runtime.Engine(d, max_prefill_tokens=32768, max_decode_batch=max_dec, n_pages=n * pages + 64, n_slots=n + 8,
                     max_pages_per_slot=pages + 1, max_out=out + 1)
print(f"init {time.time() - t0:.1f}s", flush=True)
for rate in rates:
    arr = "zero" if rate == "inf" else f"poisson:{rate}"
    base = f"n={n};input={inp};output={out};seed=1;arrival={arr};kv_capacity_blocks={n * pages + 64}"
    for spec in sys.argv[1:]:
        full = f"{base};{spec}"
        eng.run(full)
        for _ in range(reps):
            w0 = time.time()
            r = eng.run(full)
            rep = r.report
            print(f"rate {rate:>5s} {rep['tokens_per_s']:9.1f} tok/s ttft50 {1e3 * rep['p50_ttft_s']:8.1f} ms "
                  f"tbt50 {1e3 * rep['p50_tbt_s']:7.2f} ms makespan {rep['makespan_s']:.3f}s wall {time.time() - w0:.1f}s | {spec}",
                  flush=True)
eng.close()

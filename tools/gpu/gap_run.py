import os, sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, os.getcwd())
import bench
from oracle import model as M
from paper_2505_03763_b200 import runtime
w = dict(bench.WORKLOADS["1b"])
desc = M.LLAMA_1B
pages_per = (512 + 128 + 15) // 16
w["kv_pages"] = w["n"] * pages_per + 64
eng = runtime.Engine(desc, max_prefill_tokens=w["max_prefill"], max_decode_batch=w["max_decode"], n_pages=w["kv_pages"],
                     n_slots=w["n"] + 8, max_pages_per_slot=pages_per + 1, max_out=w["output"] + 1)
spec = bench.spec_for(w, "policy=sequential;max_batch=64;engine.split=0", 0, 1)
eng.run(spec); eng.run(spec)
os.makedirs("gpurun_out/gap", exist_ok=True)
eng.run(spec + ";output_dir=gpurun_out/gap;emit_event_log=1")
eng.close()

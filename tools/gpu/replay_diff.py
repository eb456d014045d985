"""Find a GPU run whose events.csv the reference replays to a different report (debug)."""
import os, shutil, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import model as M
from paper_2505_03763_b200 import runtime
eng = runtime.Engine(M.TINY, max_prefill_tokens=1024, max_decode_batch=16, n_pages=512, n_slots=16,
                     max_pages_per_slot=8, max_out=40)
for i in range(20):
    d = tempfile.mkdtemp()
    eng.run("n=8;input=64;output=32;seed=1;kv_capacity_blocks=480;policy=pipelined_splitwiser;P=2;max_batch=4;"
            f"engine.split=1;output_dir={d};emit_event_log=1")
    subprocess.run(["oracle/_ref/refwrite", "--replay", f"{d}/events.csv"], check=True)
    a = open(f"{d}/report.json").read(); b = open(f"{d}/replay_report.json").read()
    if a != b:
        os.makedirs("gpurun_out/replay_diff", exist_ok=True)
        for f in ("events.csv", "report.json", "replay_report.json"):
            shutil.copy(f"{d}/{f}", f"gpurun_out/replay_diff/{f}")
        print("mismatch at run", i)
        break
else:
    print("no mismatch in 20 runs")
eng.close()

import sys; sys.path.insert(0,'/root/repo')
from oracle import model as M
from paper_2505_03763_b200 import runtime
e = runtime.Engine(M.TINY, max_prefill_tokens=4096, max_decode_batch=64, n_pages=4096, n_slots=128, max_pages_per_slot=64, max_out=260)
for spec in ["n=96;input=16..500;output=2..40;seed=3;arrival=poisson:300;policy=mixed_batching;engine.split=1",
             "n=96;input=16..500;output=2..40;seed=3;arrival=poisson:300;policy=continuous_batching;engine.split=0"]:
    r = e.run(spec)
    err = r.extra.get("report_error")
    print(spec[-40:], "ERR" if err else "ok", err)
    if err:
        lines = r.event_log.splitlines()
        arr = {}
        for l in lines[2:]:
            t, k, d = l.split(",", 2)
            kv = dict(x.split("=",1) for x in d.split(";") if "=" in x)
            if k == "arrival": arr[int(kv["req"])] = float(t)
        bd = {}
        for l in lines[2:]:
            t, k, d = l.split(",", 2)
            kv = dict(x.split("=",1) for x in d.split(";") if "=" in x)
            if k == "batch_def": bd[int(kv["batch"])] = [int(x) for x in kv["reqs"].split("|")]
            if k == "task_start" and kv.get("kind") == "prompt":
                for rid in bd[int(kv["batch"])]:
                    if arr.get(rid, 1e9) > float(t):
                        print("  prompt start", t, "before arrival of", rid, arr.get(rid))
                        break

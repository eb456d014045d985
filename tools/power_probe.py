"""Is phase concurrency on one B200 bounded by power?  Runs, each for ~3 s of
back-to-back work while nvidia-smi samples SM clock, power and throttle
reasons: a Llama-8B prefill (8 x 1024 tokens) on the whole GPU and on a
100-SM green partition, a read stream (torch reduction over 4 GB) on the other
48 SMs, both at once, and a pure FMA spin on 48 SMs beside the prefill (no
memory traffic).  Reports work rate, median SM MHz and power per case.

  python tools/power_probe.py [--decode-sms 48]
"""
import argparse
import ctypes
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2505_03763_b200 as sw
from paper_2505_03763_b200 import runtime, shapes
from oracle import model as M


class Sampler:
    def __init__(self):
        self.s, self._stop = [], threading.Event()

    def __enter__(self):
        def loop():
            q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown"
            while not self._stop.is_set():
                out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True).stdout.strip()
                if out:
                    self.s.append([x.strip() for x in out.split(",")])
                self._stop.wait(0.1)

        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()

    def summary(self):
        mhz = [float(x[0]) for x in self.s if x[0].replace(".", "").isdigit()]
        pw = [float(x[1]) for x in self.s if x[1].replace(".", "").isdigit()]
        cap = sum(1 for x in self.s if len(x) > 2 and x[2].lower() == "active")
        return f"SM {np.median(mhz):6.0f} MHz, power {np.median(pw):5.0f} W, power-cap active {cap}/{len(self.s)}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--decode-sms", type=int, default=48)
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    d = shapes.LLAMA_8B
    P, Sp = 8, 1024
    pages = (Sp + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=P * Sp, max_decode_batch=8, n_pages=P * pages + 8, n_slots=P,
                         max_pages_per_slot=pages, max_out=4)
    L = sw.lib()
    ptoks = np.concatenate([M.prompt_tokens(d.seed, i, Sp, d.vocab) for i in range(P)])
    keep = [(ctypes.c_int32 * P)(*range(P)), (ctypes.c_int32 * P)(*([Sp] * P)),
            (ctypes.c_int32 * len(ptoks))(*ptoks.tolist()),
            (ctypes.c_int32 * (P * pages))(*range(P * pages)), (ctypes.c_int32 * P)(*([0] * P))]
    pb = sw.Batch(n=P, slots=keep[0], n_tokens=keep[1], tokens=keep[2], page_rows=keep[3], out_index=keep[4])
    dp, pp, dn, pn = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int(), ctypes.c_int()
    sw.check(L.sw_sm_partition(0, args.decode_sms, ctypes.byref(dp), ctypes.byref(pp), ctypes.byref(dn), ctypes.byref(pn)))
    full = torch.cuda.Stream()
    buf = torch.empty((4 << 30) // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty(1, device="cuda")
    spin_x = torch.randn(dn.value * 4 * 1024, device="cuda")

    def prefill(st):
        sw.check(L.sw_prefill_enqueue(eng.model, eng.kv, ctypes.byref(pb), ctypes.c_void_p(st)))

    def stream(st):
        with torch.cuda.stream(torch.cuda.ExternalStream(st)):
            torch.sum(buf, dim=0, out=sink[0])

    def spin(st):  # FMA-bound elementwise chain on a small resident tensor (no HBM traffic to speak of)
        with torch.cuda.stream(torch.cuda.ExternalStream(st)):
            y = spin_x
            for _ in range(50):
                y = torch.addcmul(y, y, y, value=1e-6)

    def run(name, jobs):
        """jobs: list of (fn, stream, work per launch, unit, launches per round); every round enqueues each
        job's launches on its own stream, then synchronizes.  Returns seconds per launch of each job."""
        for fn, st, _, _, _ in jobs:
            fn(st)
        torch.cuda.synchronize()
        counts = [0] * len(jobs)
        t0 = time.time()
        with Sampler() as smp:
            while time.time() - t0 < args.seconds:
                for i, (fn, st, _, _, reps) in enumerate(jobs):
                    for _ in range(reps):
                        fn(st)
                    counts[i] += reps
                torch.cuda.synchronize()
                if not jobs:
                    time.sleep(0.1)
            dt = time.time() - t0
        rates = ", ".join(f"{c * w / dt / (1e12 if u == 'TFLOP/s' else 1e9):.0f} {u}" for c, (_, _, w, u, _) in
                          zip(counts, jobs))
        print(f"{name:<44s} {rates:<40s} {smp.summary()}", flush=True)
        return [dt / max(c, 1) for c in counts]

    flops = 2.0 * P * Sp * (d.n_layers * (d.d_model * (d.n_heads + 2 * d.n_kv_heads) * d.head_dim +
                                          d.n_heads * d.head_dim * d.d_model + 3 * d.d_model * d.ffn_dim))
    gb = float(buf.numel() * 4)
    print(f"decode partition {dn.value} SMs, prefill partition {pn.value} SMs", flush=True)
    run("idle", [])
    run("prefill, whole GPU", [(prefill, full.cuda_stream, flops, "TFLOP/s", 1)])
    t_pre = run(f"prefill, {pn.value} SMs", [(prefill, pp.value, flops, "TFLOP/s", 1)])[0]
    t_str = run(f"stream, {dn.value} SMs", [(stream, dp.value, gb, "GB/s", 4)])[0]
    run("stream, whole GPU", [(stream, full.cuda_stream, gb, "GB/s", 4)])
    t_spin = run(f"FMA spin, {dn.value} SMs", [(spin, dp.value, 0.0, "GB/s", 2)])[0]
    run(f"prefill {pn.value} SMs + stream {dn.value} SMs",
        [(prefill, pp.value, flops, "TFLOP/s", 1), (stream, dp.value, gb, "GB/s", max(1, round(t_pre / t_str)))])
    run(f"prefill {pn.value} SMs + FMA spin {dn.value} SMs",
        [(prefill, pp.value, flops, "TFLOP/s", 1), (spin, dp.value, 0.0, "GB/s", max(1, round(t_pre / t_spin)))])
    eng.close()


if __name__ == "__main__":
    main()

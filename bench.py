"""Benchmark: split-phase vs serial tokens/s on one B200 (and request-sharded
replicas on N GPUs), with p50 TTFT/TBT, a whole-run roofline, kernel roofline
lines and the CPU oracle timed beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]

A "step" is one complete engine run of the workload through the C-ABI
(sw_engine_run).  The default workload is BASELINE.json configs[2] as SURVEY.md
§8d states it -- the Llama-3-8B shape the north-star target is quoted on:
bf16 random weights, 512 requests, prompts U[128,2048], 256 generated tokens,
Poisson arrivals at a rate where arrivals no longer limit throughput (the rate
sweep is in profiles/r02/).  Split = MixedBatching (one prompt task and one token
step in flight together) with the phases on concurrent streams / SM partitions;
serial = ContinuousBatching (the fastest serial schedule of this trace) with
every task on one stream.  value = generated tokens / device makespan (CUDA
events inside the engine) over the K timed runs; e2e = the same tokens over the
wall time of the sw_engine_run calls (prompt H2D staging and token/page-table
D2H inside).  Under torchrun every rank runs its own engine on its round-robin
shard of an N x 512-request trace (weak scaling); the per-request results are
gathered with one NCCL all_gather (paper_2505_03763_b200/sharded.py) and folded
into global percentiles; device times are the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s/GPU split vs serial prefill+decode; p50 TTFT and TBT; 1/2/4/8 GPU"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

WORKLOADS = {
    # configs[2] of BASELINE.json, as SURVEY.md §8d states it -- the default line: 8B shape, 512 requests,
    # prompts U[128,2048], 256 generated, Poisson arrivals; MixedBatching split vs ContinuousBatching serial
    "8b-cfg3": dict(model="LLAMA_8B", n=512, input="128..2048", output=256, arrival="poisson:128",
                    max_prefill=32768, max_decode=256,
                    split="policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1",
                    serial="policy=continuous_batching;max_batch=256;engine.split=0",
                    best_serial=None,
                    # chunked prefill, 8192-token chunks fused with the token step
                    # (profiles/r02s4/cfg3_chunked_sweep.txt: the best throughput of the budgets swept)
                    chunked="policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1",
                    dominant="attention"),
    # configs[1] of BASELINE.json
    # split = PipelinedSplitwiser P=2 on concurrent streams (token steps of the two lanes aligned and merged);
    # serial = the SAME task stream under the one-task gate; best_serial = the fastest
    # serial policy on this closed batch (request-level batching of all 64), reported beside it
    "1b": dict(model="LLAMA_1B", n=64, input=512, output=128, arrival="zero", max_prefill=32768, max_decode=64,
               # prefill stream at the higher priority: on this closed batch the prompt sharing the GPU with
               # the first lane's steps should finish first, so both lanes' steps merge sooner
               # (profiles/r01c/priority_1b_8b.txt: 241.1 -> 231.8 ms per run)
               split="policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.prefill_priority=1",
               serial="policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=0",
               best_serial="policy=sequential;max_batch=64;engine.split=0"),
    # configs[2]: 8B shape, Poisson arrivals of mixed prompts, mixed batching vs continuous batching
    "8b-poisson": dict(model="LLAMA_8B", n=128, input="128..2048", output=256, arrival="poisson:32",
                       max_prefill=32768, max_decode=128,
                       # prefill || decode, one instance; the prefill stream outranks the decode stream:
                       # with decode first, back-to-back PDL-chained steps starve the prompts (p50 TTFT 1.38 s,
                       # 5264 tok/s; profiles/r02s4/poisson32_priority.txt)
                       split="policy=mixed_batching;max_batch=128;engine.split=1;engine.prefill_priority=1",
                       serial="policy=mixed_batching;max_batch=128;engine.split=0",
                       best_serial="policy=continuous_batching;max_batch=128;engine.split=0"),
    # configs[4]: 8B long-context decode-heavy, prompt 8192 / gen 512, the KV arena near HBM capacity
    # (112 requests x 544 pages x 2 MiB = 128 GB of KV next to 16 GB of weights); AllAtZero
    "8b-long": dict(model="LLAMA_8B", n=112, input=8192, output=512, arrival="zero", max_prefill=32768,
                    max_decode=112,
                    split="policy=mixed_batching;max_batch=112;engine.split=1",
                    serial="policy=continuous_batching;max_batch=112;engine.split=0",
                    best_serial="policy=sequential;max_batch=112;engine.split=0",
                    # chunked prefill: p50 TTFT 12.8 -> 6.8 s at 0.99x (profiles/r02s4/bench_8b_long_chunked16384.jsonl)
                    chunked="policy=chunked_prefill;max_batch=112;chunk_tokens=16384;engine.split=1;engine.fuse=1",
                    dominant="attention"),
    # configs[0] shape on the GPU (fast sanity run)
    "tiny": dict(model="TINY", n=8, input=64, output=32, arrival="zero", max_prefill=1024, max_decode=16,
                 split="policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=1",
                 serial="policy=pipelined_splitwiser;P=2;max_batch=4;engine.split=0",
                 best_serial="policy=sequential;max_batch=8;engine.split=0"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU oracle
def cpu_sample(desc_name: str, n_req: int = 4, prompt: int = 512, gen: int = 8):
    """Time the fp32 CPU oracle (oracle/model.py, numpy/BLAS on all host
    threads) on a bounded sample of the workload: n_req requests of the same
    prompt length, `gen` greedy tokens each (x_1 from the prompt pass, then
    gen-1 batched decode steps).  Weight generation is excluded."""
    import numpy as np
    from oracle import model as M

    desc = getattr(M, desc_name)
    t_init = time.perf_counter()
    o = M.OracleModel(desc)
    t_init = time.perf_counter() - t_init
    prompts = [M.prompt_tokens(desc.seed, r, prompt, desc.vocab) for r in range(n_req)]
    rows = [list(range(64 * r, 64 * r + 64)) for r in range(n_req)]
    t0 = time.perf_counter()
    lg = o.prefill(prompts, rows)
    toks = [int(np.argmax(l)) for l in lg]
    for g in range(1, gen):
        lg = o.decode(toks, [prompt + g - 1] * n_req, rows)
        toks = [int(np.argmax(l)) for l in lg]
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": n_req * gen / dt, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"{desc_name} full depth fp32 numpy oracle: {n_req} requests x prompt {prompt}, {gen} greedy "
                      f"tokens each (prompt pass + {gen - 1} batched decode steps); weight init {t_init:.1f}s excluded",
            "seconds": dt}


def reference_simulator(w: dict, kv_pages: int) -> dict | None:
    """The unmodified reference simulator (oracle/_ref/refsim, compiled from the
    reference's own headers) on the same trace and policies: its wall time is the
    reference's scheduling-only cost of the path, and its report is what the
    reference's roofline pricing predicts for split vs serial (on its modelled
    GPU, not a B200).  Engine-only keys (engine.*) are stripped; None when the
    binary is absent."""
    exe = os.path.join(ROOT, "oracle", "_ref", "refsim")
    if not os.access(exe, os.X_OK):
        return None
    out = {"binary": "oracle/_ref/refsim (reference splitsim headers, unmodified)"}
    for arm in ("split", "serial"):
        items = [x for x in w[arm].split(";") if x]
        pol = ";".join(x for x in items if not x.startswith("engine."))
        if "policy=pipelined_splitwiser" in items:  # multi-lane: the reference's concurrent (MPS) law for the
            # split arm, its time-sliced law (one lane's task at a time) for the one-stream serial arm
            pol += ";mode=mps_concurrent" if "engine.split=1" in items else ";mode=time_sliced"
        spec = (f"n={w['n']};input={w['input']};output={w['output']};seed=1;arrival={w['arrival']};"
                f"kv_capacity_blocks={kv_pages};{pol}")
        t0 = time.perf_counter()
        try:
            r = subprocess.run([exe, spec], capture_output=True, text=True, timeout=120)
        except (OSError, subprocess.TimeoutExpired) as e:  # never fail the bench line on the reference leg
            return dict(out, error=f"refsim: {e}")
        wall = time.perf_counter() - t0
        rep = next((l for l in r.stdout.splitlines() if l.startswith("#report ")), None)
        if r.returncode != 0 or rep is None:
            return dict(out, error=f"refsim exit {r.returncode}: {r.stderr.strip()[:200]}")
        kv = dict(x.split("=", 1) for x in rep[len("#report "):].split(";") if "=" in x)
        out[arm] = {"policy": pol, "wall_s": round(wall, 4), "simulated_tokens_per_s": round(float(kv["tokens_per_s"]), 1)}
    out["simulated_split_over_serial"] = round(out["split"]["simulated_tokens_per_s"] /
                                               out["serial"]["simulated_tokens_per_s"], 4)
    return out


# ----------------------------------------------------------------- roofline
def graph_time(launch, reps: int) -> float:
    """Average device time of one launch: `reps` launches captured in one CUDA
    graph (no host launch gaps between them), replayed once to warm, then timed
    with CUDA events on the replay stream."""
    import torch

    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            launch(i)
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def roofline_decode_gemm(eng, desc, rows: int, peaks, reps: int = 20):
    """The dominant kernel: the decode step's gate/up projection (swap-AB
    tcgen05 GEMM with fused SwiGLU), HBM-bound.  Timed with CUDA events on the
    stream it is launched on (captured in a CUDA graph), rotating over all layers' weights (> L2) so every
    launch streams from HBM.  Algorithmic bytes per launch = weights 2*ffn*d*2 +
    activations rows*d*2 in + rows*ffn*2 out."""
    import ctypes
    import torch
    import paper_2505_03763_b200 as sw

    d, F, L = desc.d_model, desc.ffn_dim, desc.n_layers
    x = torch.randn(rows, d, device="cuda").bfloat16()
    y = torch.empty(rows, F, device="cuda", dtype=torch.bfloat16)
    ws = [eng.tensor(f"layer{l}.wgu")[0] for l in range(L)]
    def launch(i):
        sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ws[i % L]),
                                     ctypes.c_void_p(y.data_ptr()), rows, 2 * F, d, 2,
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

    for i in range(L):
        launch(i)
    t = graph_time(launch, reps)
    nbytes = 2 * F * d * 2 + rows * d * 2 + rows * F * 2
    achieved = nbytes / t / 1e9
    peak = float(peaks["hbm_gbs"])
    form = ("gemm_dsk_kernel<256,SWIGLU> (decode gate/up: whole tiles per SM + stream-K remainder, rows=%d)" % rows
            if rows > 128 and 2 * F // 128 > torch.cuda.get_device_properties(0).multi_processor_count else
            "gemm_decode_kernel<BN,SWIGLU> (decode gate/up, cluster split-K, rows=%d)" % rows)
    # at 256 rows the launch sits at the ridge point (2*rows FLOP per weight byte = 256 FLOP/B against
    # 1650.6 TFLOP/s / 6449 GB/s = 256): the tensor fraction is reported beside the HBM one
    flops = 2.0 * rows * 2 * F * d
    tpeak = float(peaks["bf16_tflops"])
    return {"kernel": form, "bound": "hbm",
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "bytes_per_launch": nbytes, "us_per_launch": round(t * 1e6, 2),
            "flops_per_launch": flops, "tensor_tflops": round(flops / t / 1e12, 1),
            "tensor_frac": round(flops / t / 1e12 / tpeak, 4)}


def roofline_decode_attention(eng, desc, rows: int, ctx: int, peaks, reps: int = 5, prefilled: bool = False,
                              settle_s: float = 0.0):
    """The dominant kernel of the decode-heavy 8B runs (the launch lists in profiles/r02s4: ~52% of a
    b = 256 decode step, the largest kernel class of configs[2]): paged-KV decode attention.  `rows`
    synthetic prompts of `ctx` tokens are prefilled into the arena, then one step's attention -- every
    layer's launch of the kernel the step picks -- runs back to back through sw_op_decode_attention,
    timed with CUDA events on the launching stream.  Algorithmic bytes per layer launch = the rows'
    K and V pages (rows * (ctx + 1) * 2 * Hkv * hd * 2) + q in and attention out (rows * H * hd * 2 each)."""
    import ctypes
    import numpy as np
    import torch
    import paper_2505_03763_b200 as sw

    per = (ctx + 1 + 15) // 16
    pages = [[i * per + j for j in range(per)] for i in range(rows)]
    chunk = max(1, 32768 // ctx)
    for c0 in ([] if prefilled else range(0, rows, chunk)):
        idx = list(range(c0, min(rows, c0 + chunk)))
        prompts = [np.arange(ctx, dtype=np.int64) * 7919 % desc.vocab for _ in idx]
        eng.prefill(idx, prompts, [pages[i][:(ctx + 15) // 16] for i in idx], logits=False)
    torch.cuda.synchronize()
    keep = []

    def arr(xs):
        a = (ctypes.c_int32 * len(xs))(*[int(v) for v in xs])
        keep.append(a)
        return a

    b = sw.Batch(n=rows, slots=arr(range(rows)), positions=arr([ctx] * rows))
    b.new_page = arr([pages[i][ctx // 16] if ctx % 16 == 0 else -1 for i in range(rows)])
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    lib = sw.lib()
    nbytes = rows * (ctx + 1) * 2 * desc.n_kv_heads * desc.head_dim * 2 + 2 * rows * desc.n_heads * desc.head_dim * 2
    peak = float(peaks["hbm_gbs"])

    def timed():
        for _ in range(2):
            sw.check(lib.sw_op_decode_attention(eng.model, eng.kv, ctypes.byref(b), sp))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            e0.record(st)
            for _ in range(reps):
                sw.check(lib.sw_op_decode_attention(eng.model, eng.kv, ctypes.byref(b), sp))
            e1.record(st)
            torch.cuda.synchronize()
        t_layer = e0.elapsed_time(e1) / 1e3 / reps / desc.n_layers
        return t_layer, clk.summary()["sm_mhz"]

    # first right after the prefill that filled the arena (the board power-capped, as inside a run), then
    # after `settle_s` idle: the kernel timed alone, the conditions of the burst peak it is divided by.
    # The kernel is SM-clock sensitive (per-unit prologue/merge latency chains): profiles/r02s5/attn_clock.txt
    t_hot, mhz_hot = timed()
    t_layer, mhz = t_hot, mhz_hot
    if settle_s:
        time.sleep(settle_s)
        t_layer, mhz = timed()
    achieved = nbytes / t_layer / 1e9
    out = {"kernel": f"attn_decode (paged-KV decode attention, {rows} rows x ctx {ctx + 1}, per layer)",
           "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "bytes_per_launch": nbytes, "us_per_launch": round(t_layer * 1e6, 2),
           "sm_mhz": mhz, "frac_of_8tbs_spec": round(achieved / 8000.0, 4),
           "peak_note": "peak = MEASURED_PEAKS hbm_gbs, a copy (read+write) rate; this kernel is a read stream, "
                        "which the DRAM sustains above the copy rate (ncu: 6.87 TB/s DRAM read at 1.79 GHz, "
                        "profiles/r02s4/decode_attention_ncu_full.txt), so frac can exceed 1; frac_of_8tbs_spec "
                        "is against the ~8 TB/s the north star quotes"}
    if settle_s:
        out["conditions"] = f"timed alone after {settle_s:g} s idle (burst conditions)"
        out["after_prefill"] = {"us_per_launch": round(t_hot * 1e6, 2), "achieved": round(nbytes / t_hot / 1e9, 1),
                                "frac": round(nbytes / t_hot / 1e9 / peak, 4), "sm_mhz": mhz_hot,
                                "conditions": "timed right after the arena's prefill (board at its power cap)"}
    return out


def roofline_prefill_gemm(eng, desc, tokens: int, peaks, reps: int = 10):
    """Prefill gate/up projection (normal-mode tcgen05 GEMM on CTA pairs + SwiGLU), tensor-bound."""
    import ctypes
    import torch
    import paper_2505_03763_b200 as sw

    d, F, L = desc.d_model, desc.ffn_dim, desc.n_layers
    x = torch.randn(tokens, d, device="cuda").bfloat16()
    y = torch.empty(tokens, F, device="cuda", dtype=torch.bfloat16)
    ws = [eng.tensor(f"layer{l}.wgu")[0] for l in range(L)]
    def launch(i):
        sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(ws[i % L]),
                                     ctypes.c_void_p(y.data_ptr()), tokens, 2 * F, d, 2,
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

    launch(0)
    t = graph_time(launch, reps)
    flops = 2.0 * tokens * 2 * F * d
    achieved = flops / t / 1e12
    # timed alone (10 launches, ~10 ms): the burst peak (MEASURED_PEAKS bf16_tflops, cuBLAS best of 10)
    peak = float(peaks["bf16_tflops"])
    return {"kernel": "gemm_tc_kernel<256,SWIGLU,normal,pair> (prefill gate/up, CTA-pair cta_group::2, tokens=%d)" % tokens,
            "bound": "tensor",
            "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
            "us_per_launch": round(t * 1e6, 1)}


# ----------------------------------------------------------------- engine runs
# bounded CPU samples of each model (requests, prompt, generated tokens): ~10-30 s of numpy on the host cores
CPU_SAMPLE = {"LLAMA_8B": (2, 512, 4), "LLAMA_1B": (4, 512, 8), "TINY": (8, 64, 32)}


def global_arrival(arrival: str, world: int) -> str:
    """Weak scaling: every GPU sees the single-GPU workload -- `n` requests at the
    workload's rate.  The global trace therefore has n * world requests arriving
    world times as fast; its round-robin shards (`shard=r/N`, the reference's
    multi_instance_split) each carry the per-GPU rate.  With the rate left global,
    each shard would see rate / world and the run would turn arrival-bound as N
    grows (configs[2] at 16 requests/s per GPU: 4.3k instead of 9.6k tok/s)."""
    if world <= 1:
        return arrival
    if arrival.startswith("poisson:"):
        return f"poisson:{float(arrival[len('poisson:'):]) * world:g}"
    if arrival.startswith("fixed:"):
        return f"fixed:{float(arrival[len('fixed:'):]) / world:g}"
    return arrival  # all at zero


def spec_for(w, extra: str, rank: int, world: int) -> str:
    s = (f"n={w['n'] * world};input={w['input']};output={w['output']};seed=1;"
         f"arrival={global_arrival(w['arrival'], world)};kv_capacity_blocks={w['kv_pages']};{extra}")
    if world > 1:
        s += f";shard={rank}/{world}"
    return s


def gather_run_stats(dist, world: int, res: dict, device) -> dict:
    """Scalar gather across request-sharded replicas (NCCL over NVLink on the
    GPU box, gloo in the CPU tests): makespan and wall are the max over ranks,
    tokens the sum."""
    import torch

    t = torch.tensor([res["makespan"], res["wall"], float(res["tokens"])], device=device, dtype=torch.float64)
    g = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(g, t)
    out = dict(res)
    out["makespan"] = max(float(x[0]) for x in g)
    out["wall"] = max(float(x[1]) for x in g)
    out["tokens"] = sum(float(x[2]) for x in g)
    return out


def run_work(event_log: str):
    """Algorithmic work of one run from its event log: the GPU executor prices
    every prompt task with its prefill FLOPs and every token step with its
    decode bytes (engine/gpu_executor.cu ModelWork)."""
    flops = nbytes = 0.0
    for line in event_log.splitlines():
        if ",task_start," not in line:
            continue
        kv = dict(x.split("=", 1) for x in line.split(",", 2)[2].split(";") if "=" in x)
        if kv.get("kind") == "prompt":
            flops += float(kv["compute"])
        else:
            nbytes += float(kv["mem"])
    return flops, nbytes


def run_many(eng, spec: str, k: int):
    import paper_2505_03763_b200 as sw
    from paper_2505_03763_b200 import sharded

    runs = []
    l0 = sw.launch_count()
    h0, d0 = sw.transfer_bytes()
    for _ in range(k):
        t0 = time.perf_counter()
        r = eng.run(spec)
        wall = time.perf_counter() - t0
        runs.append({"tokens": int(r.report["total_output_tokens"]), "makespan": r.report["makespan_s"], "wall": wall,
                     "rows": sharded.request_rows(r), "work": run_work(r.event_log), "report": r.report})
    h1, d1 = sw.transfer_bytes()
    return dict(runs=runs, launches=sw.launch_count() - l0, h2d=(h1 - h0) / max(k, 1), d2h=(d1 - d0) / max(k, 1))


def fold_runs(res: dict, dist, world: int, device, n_local: int, max_out: int) -> dict:
    """Per run: gather every rank's request rows (one all_gather, after the
    timed region) and fold them into global metrics; then sum tokens and device
    makespans over the K runs and take the median of the per-run percentiles."""
    from paper_2505_03763_b200 import sharded

    folds, tokens, makespan, wall = [], 0, 0.0, 0.0
    for run in res["runs"]:
        if dist:
            rows, mk, wl = sharded.gather_requests(dist, world, run["rows"], run["makespan"], run["wall"], device,
                                                   n_local + 8, max_out)
        else:
            rows, mk, wl = run["rows"], run["makespan"], run["wall"]
        f = sharded.fold(rows, mk)
        folds.append(f)
        tokens += f["total_output_tokens"]
        makespan += mk
        wall += wl
    med = lambda key: statistics.median(f[key] for f in folds)  # noqa: E731
    return dict(tokens=tokens, makespan=makespan, wall=wall, p50_ttft=med("p50_ttft_s"), p50_tbt=med("p50_tbt_s"),
                p99_tbt=med("p99_tbt_s"), n_requests=folds[-1]["n_requests"], launches=res["launches"],
                h2d=res["h2d"], d2h=res["d2h"], work=res["runs"][-1]["work"], last_tokens=res["runs"][-1]["tokens"],
                last_makespan=res["runs"][-1]["makespan"])


def whole_run_roofline(res: dict, peaks) -> dict:
    """F = sum of prefill FLOPs, B = sum of decode bytes of the
    run; serial bound t_s = F/P_tc + B/BW, split bound t_p = max(F/P_tc, B/BW);
    achieved = the run's makespan against them (P_tc the sustained bf16 peak:
    a run is a long step)."""
    F, B = res["work"]
    p_tc = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])) * 1e12
    bw = float(peaks["hbm_gbs"]) * 1e9
    t_s, t_p = F / p_tc + B / bw, max(F / p_tc, B / bw)
    toks, mk = res["last_tokens"], res["last_makespan"]
    return {"prefill_tflop": round(F / 1e12, 2), "decode_gb": round(B / 1e9, 2), "tokens": toks,
            "serial_bound_tok_s": round(toks / t_s, 1), "split_bound_tok_s": round(toks / t_p, 1),
            "achieved_tok_s": round(toks / mk, 1), "frac_of_serial_bound": round(t_s / mk, 4),
            "frac_of_split_bound": round(t_p / mk, 4), "max_split_speedup": round(t_s / t_p, 4),
            "peaks": {"tensor_tflops": p_tc / 1e12, "hbm_gbs": bw / 1e9}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="8b-cfg3")
    ap.add_argument("--split", default=None, help="override the split-phase policy spec")
    ap.add_argument("--serial", default=None, help="override the serial policy spec")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = dict(WORKLOADS[args.workload])
    peaks, peaks_src = load_peaks()

    if args.impl == "reference":
        # The reference's own CPU implementation of the path: it has no model math
        # (splitsim prices phases with a roofline law), so this arm times the fp32
        # CPU oracle port on the host cores, rank 0 only, on a bounded sample of
        # this workload's model.
        if rank != 0:
            return
        n_req, prompt, gen = CPU_SAMPLE[w["model"]]
        samples = [cpu_sample(w["model"], n_req, prompt, gen) for _ in range(max(args.steps, 1))]
        v = statistics.median(s["value"] for s in samples)
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": 0, "ms_per_step": round(1e3 * statistics.median(s["seconds"] for s in samples), 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": args.workload, "model_shape": w["model"], "sample": samples[0]["sample"]},
                "cpu_baseline": {k: samples[0][k] for k in ("unit", "cores", "kind", "sample")} | {"value": round(v, 3)},
                "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        in_max = int(str(w["input"]).split("..")[-1])
        line["reference_simulator"] = reference_simulator(w, w["n"] * ((in_max + w["output"] + 15) // 16) + 64)
        print(json.dumps(line), flush=True)
        return

    import torch

    # SW_BENCH_BACKEND=gloo: the multi-rank path with every rank on the visible GPUs round robin and the
    # gather on host tensors -- a functional check of the N > 1 line on a one-GPU box (tests, not timing)
    backend = os.environ.get("SW_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2505_03763_b200 import runtime, shapes

    desc = getattr(shapes, w["model"])
    n_local = w["n"]
    in_max = int(str(w["input"]).split("..")[-1])
    pages_per = (in_max + w["output"] + 15) // 16
    t_init = time.perf_counter()
    # KV arena: the trace's worst case, capped by what fits in free HBM (sw_kv_capacity_pages)
    eng = runtime.Engine(desc, max_prefill_tokens=w["max_prefill"], max_decode_batch=w["max_decode"],
                         n_pages=None, n_slots=n_local + 8, max_pages_per_slot=pages_per + 1,
                         max_out=w["output"] + 1, device=local, kv_reserve_bytes=4 << 30,
                         max_pages=n_local * pages_per + 64)
    w["kv_pages"] = eng.n_pages
    t_init = time.perf_counter() - t_init
    split_spec = spec_for(w, args.split or w["split"], rank, world)
    serial_spec = spec_for(w, args.serial or w["serial"], rank, world)
    best_spec = spec_for(w, w["best_serial"], rank, world) if w["best_serial"] else None
    chunk_spec = spec_for(w, w["chunked"], rank, world) if w.get("chunked") else None

    for _ in range(args.warmup):
        eng.run(split_spec)
    for _ in range(max(1, args.warmup // 3)):
        eng.run(serial_spec)
        if best_spec:
            eng.run(best_spec)
        if chunk_spec:
            eng.run(chunk_spec)

    def timed(spec):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        res = run_many(eng, spec, args.steps)
        torch.cuda.synchronize()
        return res

    with ClockSampler(local) as clocks:
        split_raw = timed(split_spec)
    serial_raw = timed(serial_spec)
    best_raw = timed(best_spec) if best_spec else None
    chunk_raw = timed(chunk_spec) if chunk_spec else None
    dev = ("cuda" if backend == "nccl" else "cpu") if dist else None
    split = fold_runs(split_raw, dist, world, dev, n_local, w["output"] + 1)
    serial = fold_runs(serial_raw, dist, world, dev, n_local, w["output"] + 1)
    best = fold_runs(best_raw, dist, world, dev, n_local, w["output"] + 1) if best_raw else serial
    chunked = fold_runs(chunk_raw, dist, world, dev, n_local, w["output"] + 1) if chunk_raw else None

    roof = roofline_decode_gemm(eng, desc, w["max_decode"], peaks) if rank == 0 else None
    # decode-heavy 8B runs: the dominant kernel is the decode attention (its roofline is the line's
    # `roofline`; the decode gate/up's stays beside it as `roofline_decode_gemm`)
    roof_attn = None
    if rank == 0 and w.get("dominant") == "attention":
        in_mean = (int(str(w["input"]).split("..")[0]) + in_max) // 2
        roof_attn = roofline_decode_attention(eng, desc, w["max_decode"], in_mean + w["output"] // 2, peaks,
                                              reps=20, settle_s=3.0)
    roof_prefill = roofline_prefill_gemm(eng, desc, 4096, peaks) if rank == 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tpath) and roof:
        with open(tpath) as f:
            traffic = json.load(f).get(args.workload, {}).get("decode_gate_up_bytes")
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        eng.close()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            n_req, prompt, gen = CPU_SAMPLE[w["model"]]
            cpu = cpu_sample(w["model"], n_req, prompt, gen)
        except Exception as e:  # never fail the GPU line on the CPU sample
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}

    value = split["tokens"] / split["makespan"]
    serial_v = serial["tokens"] / serial["makespan"]
    best_v = best["tokens"] / best["makespan"]
    # decode-step roofline (closed batches): algorithmic bytes of a step at the batch and mean context of the
    # best-serial run over its p50 TBT (a step alone on the GPU)
    step = None
    if w["arrival"] == "zero" and str(w["input"]).isdigit():
        b = min(w["n"], w["max_decode"])
        ctx = int(w["input"]) + w["output"] / 2
        kv_tok = 2 * desc.n_layers * desc.n_kv_heads * desc.head_dim * 2
        n_mm = desc.n_layers * (desc.d_model * (desc.n_heads + 2 * desc.n_kv_heads) * desc.head_dim +
                                desc.n_heads * desc.head_dim * desc.d_model + 3 * desc.d_model * desc.ffn_dim)
        nbytes = 2 * (n_mm + desc.d_model * desc.vocab) + 2 * desc.d_model * b + b * ctx * kv_tok + b * kv_tok
        ach = nbytes / best["p50_tbt"] / 1e9
        step = {"rows": b, "mean_ctx": ctx, "bytes_per_step": int(nbytes), "p50_tbt_s": best["p50_tbt"],
                "achieved": round(ach, 1), "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                "frac": round(ach / float(peaks["hbm_gbs"]), 4)}
    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * split["makespan"] / args.steps, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (SplitMix64 random-init weights and prompts)",
        "config": {"workload": args.workload, "model_shape": w["model"], "requests_per_gpu": n_local,
                   "prompt": w["input"], "gen": w["output"], "arrival": w["arrival"],
                   "arrival_global": global_arrival(w["arrival"], world),
                   "split_policy": args.split or w["split"], "serial_policy": args.serial or w["serial"],
                   "best_serial_policy": w["best_serial"] or (args.serial or w["serial"]),
                   "kv_pages": w["kv_pages"],
                   "l2": "working set > L2: every decode step streams all weights (2.5-16 GB) plus the KV cache",
                   "parallelism": f"request-sharded replicas x{world}"},
        "per_gpu_tokens_per_s": round(value / world, 1),
        "split": {"tokens_per_s": round(value, 1), "p50_ttft_s": split["p50_ttft"], "p50_tbt_s": split["p50_tbt"],
                  "p99_tbt_s": split["p99_tbt"], "requests": split["n_requests"]},
        "serial": {"tokens_per_s": round(serial_v, 1), "p50_ttft_s": serial["p50_ttft"],
                   "p50_tbt_s": serial["p50_tbt"], "p99_tbt_s": serial["p99_tbt"]},
        "split_over_serial": round(value / serial_v, 4),
        "best_serial": {"tokens_per_s": round(best_v, 1), "p50_ttft_s": best["p50_ttft"], "p50_tbt_s": best["p50_tbt"]},
        "split_over_best_serial": round(value / best_v, 4),
        "chunked": ({"policy": w["chunked"], "tokens_per_s": round(chunked["tokens"] / chunked["makespan"], 1),
                     "p50_ttft_s": chunked["p50_ttft"], "p50_tbt_s": chunked["p50_tbt"], "p99_tbt_s": chunked["p99_tbt"],
                     "over_best_serial": round(chunked["tokens"] / chunked["makespan"] / best_v, 4)}
                    if chunked else None),
        "roofline_run": {"split": whole_run_roofline(split, peaks), "serial": whole_run_roofline(serial, peaks)},
        "roofline_decode_step": step,
        "e2e": {"value": round(split["tokens"] / split["wall"], 1), "unit": "tokens/s",
                "h2d_bytes_per_step": int(split["h2d"]), "d2h_bytes_per_step": int(split["d2h"])},
        "gpu_launches": int(split["launches"]),
        "roofline": None,
        "roofline_prefill": roof_prefill,
        "cpu_baseline": cpu,
        "reference_simulator": reference_simulator(w, w["kv_pages"]) if world == 1 else None,
        "clocks": clocks.summary(),
        "peaks_source": peaks_src,
        "init_s": round(t_init, 1),
    }
    if roof:
        gemm_roof = {"bound": roof["bound"], "achieved": roof["achieved"], "peak": roof["peak"],
                     "unit": roof["unit"], "frac": roof["frac"], "traffic": traffic, "kernel": roof["kernel"],
                     "us_per_launch": roof["us_per_launch"], "bytes_per_launch": roof["bytes_per_launch"],
                     "tensor_frac": roof["tensor_frac"]}
        if roof_attn:
            attn_traffic = None
            if os.path.exists(tpath):
                with open(tpath) as f:
                    attn_traffic = json.load(f).get(args.workload, {}).get("decode_attention_bytes")
            line["roofline"] = dict(roof_attn, traffic=attn_traffic)
            line["roofline_decode_gemm"] = gemm_roof
        else:
            line["roofline"] = gemm_roof
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


if __name__ == "__main__":
    main()

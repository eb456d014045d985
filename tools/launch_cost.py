"""Host cost of one decode step enqueue (StepMeta copy + CUDA graph launch) and the
in-engine per-step overhead: the stream is blocked by a long sleep kernel while K
steps are enqueued, so the host time per enqueue is measured without GPU waits.

  python tools/launch_cost.py --model LLAMA_1B --batch 64 --prompt 512
"""
import argparse, ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import model as M
import paper_2505_03763_b200 as sw
from paper_2505_03763_b200 import runtime


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="LLAMA_1B")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=512)
    args = ap.parse_args()
    d = getattr(M, args.model)
    B, S = args.batch, args.prompt
    pages_per = (S + 64 + 15) // 16
    eng = runtime.Engine(d, max_prefill_tokens=max(min(B * S, 32768), 64), max_decode_batch=B,
                         n_pages=B * pages_per + 8, n_slots=B, max_pages_per_slot=pages_per, max_out=64)
    rows = [list(range(i * pages_per, (i + 1) * pages_per)) for i in range(B)]
    prompts = [M.prompt_tokens(d.seed, i, S, d.vocab) for i in range(B)]
    eng.prefill(list(range(B)), prompts, [r[:(S + 15) // 16] for r in rows], logits=False)
    st = torch.cuda.Stream()
    slots = (ctypes.c_int32 * B)(*range(B))
    pos = (ctypes.c_int32 * B)(*([S] * B))
    newp = (ctypes.c_int32 * B)(*([-1] * B))
    b = sw.Batch(n=B, slots=slots, positions=pos)
    b.new_page = newp
    L = sw.lib()
    sp = ctypes.c_void_p(st.cuda_stream)
    with torch.cuda.stream(st):
        for _ in range(3):
            sw.check(L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(b), sp))
        torch.cuda.synchronize()
        for reps in (1, 8):
            torch.cuda._sleep(2_000_000_000 // 1000 * 50)  # ~50 ms of GPU time ahead of the enqueues
            t0 = time.perf_counter()
            for _ in range(reps):
                sw.check(L.sw_decode_enqueue(eng.model, eng.kv, ctypes.byref(b), sp))
            dt = (time.perf_counter() - t0) / reps
            torch.cuda.synchronize()
            print(f"{args.model} b={B}: host enqueue (StepMeta copy + graph launch) {dt * 1e6:.1f} us per step (x{reps})",
                  flush=True)
    eng.close()


if __name__ == "__main__":
    main()

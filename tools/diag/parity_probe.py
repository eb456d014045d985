"""Parity probe: GPU logits vs the fp32 oracle and the 16-bit-emulating oracle,
split by phase (prefill rows / decode steps) and depth; prints max/median
per-row rel-L2 and the elementwise bar |d| / max|ref_row|."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import model as M
from paper_2505_03763_b200 import runtime


def stats(a, b):
    rel = np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)
    el = np.abs(a - b).max(axis=-1) / np.abs(b).max(axis=-1)
    return f"rel max {rel.max():.4f} med {np.median(rel):.4f} | elem max {el.max():.4f}"


def run(desc, lens, steps, label):
    eng = runtime.Engine(desc, max_prefill_tokens=4096, max_decode_batch=32, n_pages=2048, n_slots=64,
                         max_pages_per_slot=128, max_out=64)
    o = M.OracleModel(desc)
    e = M.OracleModel(desc, emulate_bf16=True, share_weights_with=o)
    slots = list(range(len(lens)))
    prompts = [M.prompt_tokens(desc.seed, 100 + i, n, desc.vocab) for i, n in enumerate(lens)]
    rows = [[i * 128 + j for j in range(128)] for i in range(len(lens))]
    lg = eng.prefill(slots, prompts, [r[:(n + 15) // 16] for r, n in zip(rows, lens)])
    ref, em = o.prefill(prompts, rows), e.prefill(prompts, rows)
    print(f"{label} prefill: vs fp32 {stats(lg, ref)} || vs emu {stats(lg, em)} || emu vs fp32 {stats(em, ref)}", flush=True)
    toks = [int(np.argmax(l)) for l in ref]
    pos = list(lens)
    D32, DEM, EM32 = [], [], []
    for s in range(steps):
        newp = [rows[i][pos[i] // 16] if pos[i] % 16 == 0 else -1 for i in range(len(lens))]
        lg = eng.decode(slots, pos, tokens=toks, new_page=newp)
        ref, em = o.decode(toks, pos, rows), e.decode(toks, pos, rows)
        D32.append(lg); DEM.append(em); EM32.append(ref)
        toks = [int(np.argmax(l)) for l in ref]
        pos = [p + 1 for p in pos]
    if steps:
        g, em, ref = np.concatenate(D32), np.concatenate(DEM), np.concatenate(EM32)
        print(f"{label} decode : vs fp32 {stats(g, ref)} || vs emu {stats(g, em)} || emu vs fp32 {stats(em, ref)}", flush=True)
    eng.close()


lens = [1, 15, 16, 17, 64, 100, 129]
for L in (1, 2):
    run(dataclasses.replace(M.TINY, n_layers=L), lens, 8, f"TINY L={L}")

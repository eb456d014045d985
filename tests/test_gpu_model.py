"""Model-level parity of the CUDA path (through the C-ABI) with the CPU oracle.

Bars:
  * vs the oracle with the kernel's bf16 storage points emulated
    (emulate_bf16=True): per-row relative L2 <= 1e-2 (the north-star bar;
    what remains is accumulation order);
  * vs the pure fp32 oracle: per-row relative L2 <= 2e-2 -- bf16 activation
    rounding alone costs ~0.5-1% on these random-init models (DESIGN.md
    "Parity"), so 1e-2 is reported, not asserted, there;
  * greedy tokens identical to the fp32 oracle wherever its top-2 margin
    exceeds 1e-2 * max|logit|; page tables bit exact.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import model as M

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 1e-2       # vs emulated-format oracle
LOGIT_RTOL_FP32 = 2e-2  # vs pure fp32 oracle


def rel_rows(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def margin_tol(ref_row):
    return LOGIT_RTOL * float(np.max(np.abs(ref_row)))


@pytest.fixture(scope="module")
def tiny():
    from paper_2505_03763_b200 import runtime

    eng = runtime.Engine(M.TINY, max_prefill_tokens=2048, max_decode_batch=32, n_pages=1024, n_slots=64,
                         max_pages_per_slot=16, max_out=40)
    yield eng
    eng.close()


@pytest.fixture(scope="module")
def tiny_oracle():
    return M.OracleModel(M.TINY)


@pytest.fixture(scope="module")
def tiny_emu(tiny_oracle):
    return M.OracleModel(M.TINY, emulate_bf16=True, share_weights_with=tiny_oracle)


def test_weights_bit_exact(tiny, tiny_oracle):
    d = M.TINY
    o = tiny_oracle
    H, Hk, hd, F = d.n_heads, d.n_kv_heads, d.head_dim, d.ffn_dim
    assert np.array_equal(tiny.tensor_numpy("emb").reshape(d.vocab, d.d_model), o.emb)
    for l in range(d.n_layers):
        W = o.layers[l]
        qkv = tiny.tensor_numpy(f"layer{l}.wqkv").reshape(-1, d.d_model)
        assert np.array_equal(qkv[:H * hd], W["wq"])
        assert np.array_equal(qkv[H * hd:(H + Hk) * hd], W["wk"])
        assert np.array_equal(qkv[(H + Hk) * hd:], W["wv"])
        gu = tiny.tensor_numpy(f"layer{l}.wgu").reshape(2 * F, d.d_model)
        for j in range(F // 64):
            assert np.array_equal(gu[128 * j:128 * j + 64], W["wg"][64 * j:64 * j + 64])
            assert np.array_equal(gu[128 * j + 64:128 * j + 128], W["wu"][64 * j:64 * j + 64])
        assert np.array_equal(tiny.tensor_numpy(f"layer{l}.wo").reshape(d.d_model, -1), W["wo"])
        assert np.array_equal(tiny.tensor_numpy(f"layer{l}.wd").reshape(d.d_model, F), W["wd"])
    assert np.array_equal(tiny.tensor_numpy("lm").reshape(d.vocab, d.d_model), o.lm)


def test_prefill_then_decode_teacher_forced(tiny, tiny_oracle, tiny_emu):
    d = M.TINY
    o = tiny_oracle
    errs_fp32, errs_emu = [], []
    lens = [1, 15, 16, 17, 64, 100, 129]  # page-boundary edge cases, ragged batch
    slots = list(range(10, 10 + len(lens)))
    prompts = [M.prompt_tokens(d.seed, 100 + i, n, d.vocab) for i, n in enumerate(lens)]
    # disjoint page rows, deliberately non-contiguous ids
    rows = [[(i * 37 + j * 11) % 800 for j in range(16)] for i in range(len(lens))]
    seen = set()
    for r in rows:
        for p in r:
            assert p not in seen
            seen.add(p)
    lg = tiny.prefill(slots, prompts, [r[:(n + 15) // 16] for r, n in zip(rows, lens)])
    ref = o.prefill(prompts, rows)
    emu = tiny_emu.prefill(prompts, rows)
    errs_fp32.append(rel_rows(lg, ref))
    errs_emu.append(rel_rows(lg, emu))
    toks = [int(np.argmax(l)) for l in ref]
    for i, l in enumerate(ref):
        if M.top2_margin(l) > margin_tol(l):
            assert int(np.argmax(lg[i])) == toks[i]
    pos = list(lens)
    for step in range(20):
        newp = [rows[i][pos[i] // 16] if pos[i] % 16 == 0 else -1 for i in range(len(lens))]
        lg = tiny.decode(slots, pos, tokens=toks, new_page=newp)
        ref = o.decode(toks, pos, rows)
        emu = tiny_emu.decode(toks, pos, rows)
        errs_fp32.append(rel_rows(lg, ref))
        errs_emu.append(rel_rows(lg, emu))
        nxt = []
        for i, l in enumerate(ref):
            if M.top2_margin(l) > margin_tol(l):
                assert int(np.argmax(lg[i])) == int(np.argmax(l)), (step, i)
            nxt.append(int(np.argmax(l)))  # teacher forcing with the oracle's token
        toks = nxt
        pos = [p + 1 for p in pos]
    e32, eem = np.concatenate(errs_fp32), np.concatenate(errs_emu)
    print(f"\nlogit rel-L2 vs fp32 oracle: max {e32.max():.4f} median {np.median(e32):.4f} "
          f"frac<=1e-2 {np.mean(e32 <= 1e-2):.3f}; vs emulated-format oracle: max {eem.max():.4f}")
    assert eem.max() < LOGIT_RTOL
    assert e32.max() < LOGIT_RTOL_FP32


def test_decode_uses_device_resident_token(tiny, tiny_oracle):
    """tokens=NULL feeds last_token[slot] written by the previous launch."""
    d = M.TINY
    prompts = [M.prompt_tokens(d.seed, 300 + i, 30 + i, d.vocab) for i in range(3)]
    slots = [40, 41, 42]
    rows = [[900 + 16 * i + j for j in range(4)] for i in range(3)]
    lg = tiny.prefill(slots, prompts, [r[:2] for r in rows])
    tiny_oracle.prefill(prompts, rows)
    t1 = [int(np.argmax(l)) for l in lg]
    pos = [len(p) for p in prompts]
    lg_dev = tiny.decode(slots, pos, tokens=None, new_page=[-1] * 3)
    ref = tiny_oracle.decode(t1, pos, rows)
    assert rel_rows(lg_dev, ref).max() < LOGIT_RTOL_FP32


def _long_ctx_engine(desc, pages):
    from paper_2505_03763_b200 import runtime

    return runtime.Engine(desc, max_prefill_tokens=2048, max_decode_batch=8, n_pages=8 * pages + 8, n_slots=8,
                          max_pages_per_slot=pages, max_out=16)


@pytest.mark.parametrize("shape", ["TINY", "LLAMA_1B_2L", "LLAMA_8B_1L"])
def test_long_context_split_kv_and_split_k(shape):
    """Contexts long enough for several split-KV chunks (multi-split merge) and,
    at the 1B and 8B widths, the cluster split-K decode GEMMs: 1B runs S = 8
    (QKV, Wo, Wd) and 2 (gate/up); 8B (one layer, small vocabulary) runs the
    GPC-headroom factors S = 5 (QKV) and 7 (Wo, Wd) and S = 1 (gate/up)."""
    import dataclasses

    if shape == "TINY":
        d = M.TINY
    elif shape == "LLAMA_1B_2L":
        d = dataclasses.replace(M.LLAMA_1B, n_layers=2)
    else:
        d = dataclasses.replace(M.LLAMA_8B, n_layers=1, vocab=4096)
    pages = 80
    eng = _long_ctx_engine(d, pages)
    try:
        o = M.OracleModel(d)
        emu = M.OracleModel(d, emulate_bf16=True, share_weights_with=o)
        lens = [700, 1030] if shape != "LLAMA_8B_1L" else [300, 530]
        prompts = [M.prompt_tokens(d.seed, 500 + i, n, d.vocab) for i, n in enumerate(lens)]
        rows = [list(range(i * pages, (i + 1) * pages)) for i in range(2)]
        lg = eng.prefill([0, 1], prompts, [r[:(n + 15) // 16] for r, n in zip(rows, lens)])
        ref, em = o.prefill(prompts, rows), emu.prefill(prompts, rows)
        e32, eem = [rel_rows(lg, ref)], [rel_rows(lg, em)]
        toks = [int(np.argmax(l)) for l in ref]
        pos = list(lens)
        for _ in range(4):
            newp = [rows[i][pos[i] // 16] if pos[i] % 16 == 0 else -1 for i in range(2)]
            lg = eng.decode([0, 1], pos, tokens=toks, new_page=newp)
            ref, em = o.decode(toks, pos, rows), emu.decode(toks, pos, rows)
            e32.append(rel_rows(lg, ref))
            eem.append(rel_rows(lg, em))
            toks = [int(np.argmax(l)) for l in ref]
            pos = [p + 1 for p in pos]
        e32, eem = np.concatenate(e32), np.concatenate(eem)
        print(f"\n{shape}: rel-L2 vs fp32 max {e32.max():.4f}; vs emulated max {eem.max():.4f}")
        assert eem.max() < LOGIT_RTOL
        assert e32.max() < LOGIT_RTOL_FP32
    finally:
        eng.close()


# Llama-8B's attention geometry (head_dim 128, 4 query heads per kv head) and
# Llama-1B's (head_dim 64) at a size the oracle runs in seconds: the tcgen05
# prefill attention (head pairs), both decode-attention kernels (SW_ATTN_FLAT=0
# forces the per-unit kernel, 1 the flat one; read once per process, hence a
# child process) and the fused QKV/RoPE epilogue.
DESCS = {
    "hd128_g4": "n_layers=2, d_model=512, n_heads=8, n_kv_heads=2, head_dim=128, ffn_dim=1024, vocab=4096",
    "hd64_g4": "n_layers=2, d_model=512, n_heads=8, n_kv_heads=2, head_dim=64, ffn_dim=1024, vocab=4096",
}


@pytest.mark.parametrize("shape", sorted(DESCS))
@pytest.mark.parametrize("flat", ["0", "1"])
def test_attention_geometries_prefill_and_decode(shape, flat):
    import subprocess
    import sys
    import textwrap

    # the decode-attention choice is read once per process: run each variant in a child
    code = textwrap.dedent(f"""
        import sys, numpy as np
        sys.path.insert(0, {repr(str(__import__('pathlib').Path(__file__).resolve().parents[1]))})
        from oracle import model as M
        from paper_2505_03763_b200 import runtime
        d = M.Desc({DESCS[shape]})
        eng = runtime.Engine(d, max_prefill_tokens=4096, max_decode_batch=8, n_pages=512, n_slots=8,
                             max_pages_per_slot=40, max_out=8)
        lens = [1, 127, 128, 129, 257, 600]
        rows = [[i + 8 * j for j in range(40)] for i in range(len(lens))]
        prompts = [M.prompt_tokens(d.seed, 700 + i, n, d.vocab) for i, n in enumerate(lens)]
        lg = eng.prefill(list(range(len(lens))), prompts, [r[:(n + 15) // 16] for r, n in zip(rows, lens)])
        o = M.OracleModel(d, emulate_bf16=True)
        ref = o.prefill(prompts, [r[:(n + 15) // 16] for r, n in zip(rows, lens)])
        rel = np.linalg.norm(lg - ref, axis=1) / np.linalg.norm(ref, axis=1)
        toks = [int(np.argmax(x)) for x in ref]
        newp = [rows[i][lens[i] // 16] if lens[i] % 16 == 0 else -1 for i in range(len(lens))]
        lg2 = eng.decode(list(range(len(lens))), lens, tokens=toks, new_page=newp)
        ref2 = o.decode(toks, lens, [r[:(n + 16) // 16] for r, n in zip(rows, lens)])
        rel2 = np.linalg.norm(lg2 - ref2, axis=1) / np.linalg.norm(ref2, axis=1)
        eng.close()
        print(float(rel.max()), float(rel2.max()))
    """)
    env = dict(__import__("os").environ, SW_ATTN_FLAT=flat)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    pre, dec = map(float, p.stdout.split()[-2:])
    assert pre <= LOGIT_RTOL and dec <= LOGIT_RTOL, (pre, dec)

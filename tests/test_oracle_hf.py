"""Pin the fp32 model oracle (oracle/model.py) against an independent
implementation: HuggingFace transformers' LlamaForCausalLM (5.5, installed in
this image) loaded with the oracle's SplitMix64 weights.

The reference (splitsim) has no model math, so nothing in /root/reference can
pin the logits; this is the independent check the oracle gets instead.  Both
run in fp32 on the CPU: RMSNorm, rotate-half RoPE (theta 500000, no scaling),
GQA, SwiGLU, untied or tied LM head.  Prefill logits at every position and
incremental decode through the paged KV store must agree to fp32 accuracy.
"""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from oracle import model as M


def hf_model(o: M.OracleModel):
    from transformers import LlamaConfig, LlamaForCausalLM

    d = o.d
    cfg = LlamaConfig(vocab_size=d.vocab, hidden_size=d.d_model, intermediate_size=d.ffn_dim,
                      num_hidden_layers=d.n_layers, num_attention_heads=d.n_heads, num_key_value_heads=d.n_kv_heads,
                      head_dim=d.head_dim, rms_norm_eps=d.norm_eps, max_position_embeddings=8192,
                      rope_parameters={"rope_theta": d.rope_theta, "rope_type": "default"},
                      tie_word_embeddings=d.tied_embeddings, attention_bias=False, mlp_bias=False,
                      hidden_act="silu", torch_dtype=torch.float32)
    m = LlamaForCausalLM(cfg).float().eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(o.emb))
        for l, W in enumerate(o.layers):
            L = m.model.layers[l]
            L.self_attn.q_proj.weight.copy_(t(W["wq"]))
            L.self_attn.k_proj.weight.copy_(t(W["wk"]))
            L.self_attn.v_proj.weight.copy_(t(W["wv"]))
            L.self_attn.o_proj.weight.copy_(t(W["wo"]))
            L.mlp.gate_proj.weight.copy_(t(W["wg"]))
            L.mlp.up_proj.weight.copy_(t(W["wu"]))
            L.mlp.down_proj.weight.copy_(t(W["wd"]))
            L.input_layernorm.weight.copy_(t(o.gains["attn"][l]))
            L.post_attention_layernorm.weight.copy_(t(o.gains["mlp"][l]))
        m.model.norm.weight.copy_(t(o.gains["final"]))
        if not d.tied_embeddings:
            m.lm_head.weight.copy_(t(o.lm))
    return m


SHAPES = {
    "tiny": M.TINY,
    "1b_widths_1layer": dataclasses.replace(M.LLAMA_1B, n_layers=1, vocab=4096),
    "8b_widths_1layer": dataclasses.replace(M.LLAMA_8B, n_layers=1, vocab=4096),
}


@pytest.mark.parametrize("name", sorted(SHAPES))
def test_oracle_matches_transformers_llama(name):
    d = SHAPES[name]
    o = M.OracleModel(d)
    rng = np.random.default_rng(3)
    if name == "tiny":  # non-unit gains exercise the norm weights too
        for l in range(d.n_layers):
            o.gains["attn"][l] = M.bf16_round(rng.uniform(0.5, 1.5, d.d_model).astype(np.float32))
            o.gains["mlp"][l] = M.bf16_round(rng.uniform(0.5, 1.5, d.d_model).astype(np.float32))
        o.gains["final"] = M.bf16_round(rng.uniform(0.5, 1.5, d.d_model).astype(np.float32))
    hf = hf_model(o)
    n, steps = 40, 6
    prompt = M.prompt_tokens(d.seed, 11, n, d.vocab)
    row = list(range(8))
    # oracle: prefill logits at every prompt position, then greedy decode steps through the page store
    x = o.forward(prompt, [row], [np.arange(n)], want=np.arange(n))
    toks = [int(np.argmax(x[-1]))]
    dec = []
    for g in range(steps):
        lg = o.decode([toks[-1]], [n + g], [row])[0]
        dec.append(lg)
        toks.append(int(np.argmax(lg)))
    seq = np.concatenate([prompt, np.asarray(toks[:-1])])
    with torch.no_grad():
        ref = hf(torch.from_numpy(seq[None].astype(np.int64))).logits[0].numpy()
    mine = np.concatenate([x, np.stack(dec)])
    rel = np.linalg.norm(mine - ref, axis=1) / np.linalg.norm(ref, axis=1)
    print(f"\n{name}: oracle vs transformers LlamaForCausalLM fp32, per-row rel-L2 max {rel.max():.2e}")
    assert rel.max() < 2e-5
    assert [int(t) for t in np.argmax(ref[n - 1:], axis=1)] == toks

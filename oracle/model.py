"""ORACLE / TEST INFRASTRUCTURE ONLY -- the CPU fp32 restatement of the model math.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the timed CPU
baseline; the product path (libsplitwise.so) never calls it.

PARITY STATUS.  The reference (splitsim) has no model math at all -- a prompt
task and a token step are just (compute, mem) demands priced by a roofline law
(splitsim/gpu_model.hpp:137-189; SPEC.md:15 lists real GPU execution and model
weights as out of scope).  So this decoder is NEW, written from the north star
(RMSNorm, RoPE, GQA, SwiGLU, greedy argmax) and the phase
semantics the reference does pin:
  * a prompt task over `in` tokens writes KV[0, in) and emits no token of its
    own in the metrics (metrics.hpp:268-276); its argmax is x_1;
  * token step g feeds x_g at position in+g-1, writes that KV entry and yields
    x_{g+1}; a request gets exactly `output` steps (engine.hpp:305-310), so the
    committed output tokens are x_1..x_out and KV after step g holds in+g
    entries = blocks_for(in+g) blocks (engine.hpp:316-319);
  * KV is paged in blocks of B=16 tokens (config.hpp:33) addressed through
    per-request page tables.
No reference test pins logits or tokens; the weights/prompt generator IS
pinned to the reference's SplitMix64 (prng.hpp:10-35, checked against
oracle/_ref/refsim --prng) and the page-table layout to the reference's KV
ledger (gpu_model.hpp:79-135).  The decoder math itself is pinned against an
independent implementation instead: tests/test_oracle_hf.py loads the same
weights (and non-unit norm gains) into HuggingFace transformers'
LlamaForCausalLM and requires per-row logits within 2e-5 relative, prefill at
every position and incremental paged decode.

Synthetic inputs:
  tensor k, element i (row-major of its logical [out, in] shape):
    u = SplitMix64(seed ^ (k * 0x9E3779B97F4A7C15)).next_unit() at draw i
    w = bf16_rne(float32((2u - 1) * sqrt(3 / fan_in)))
  k = 0 embedding [V, d]; layer l: k = 1 + 7l + {0 Wq, 1 Wk, 2 Wv, 3 Wo,
  4 Wgate, 5 Wup, 6 Wdown}; k = 1 + 7L LM head (untied models).  Norm gains 1.
  prompt token j of request r = SplitMix64(seed + 1000003 r) draw j mod V.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------- SplitMix64
def splitmix_mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_at(seed: int, idx: np.ndarray) -> np.ndarray:
    """i-th draw of SplitMix64(seed) (random access form of prng.hpp:14-19)."""
    with np.errstate(over="ignore"):
        s = np.uint64(seed & MASK64) + (idx.astype(np.uint64) + np.uint64(1)) * GOLDEN
        return splitmix_mix(s)


def next_u64_stream(seed: int, n: int) -> List[int]:
    return [int(v) for v in splitmix_at(seed, np.arange(n, dtype=np.uint64))]


def f16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even IEEE half, returned as float32 values."""
    return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bfloat16, returned as float32 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


_GEN = None


def _c_gen():
    """The C restatement (oracle/gen.c) when built; identical values, ~50x faster."""
    global _GEN
    if _GEN is None:
        import ctypes
        import os

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libgen.so")
        _GEN = False
        if os.path.exists(path):
            lib = ctypes.CDLL(path)
            lib.oracle_gen_tensor.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_void_p]
            _GEN = lib
    return _GEN


def tensor_values(seed: int, k: int, rows: int, cols: int, fan_in: int, chunk: int = 1 << 24,
                  use_c: bool = True) -> np.ndarray:
    out = np.empty(rows * cols, dtype=np.float32)
    gen = _c_gen() if use_c else False
    if gen:
        gen.oracle_gen_tensor(seed & MASK64, k, rows * cols, fan_in, out.ctypes.data)
        return out.reshape(rows, cols)
    tseed = (seed ^ ((k * 0x9E3779B97F4A7C15) & MASK64)) & MASK64
    scale = math.sqrt(3.0 / fan_in)
    for s in range(0, rows * cols, chunk):
        e = min(rows * cols, s + chunk)
        u = (splitmix_at(tseed, np.arange(s, e, dtype=np.uint64)) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        out[s:e] = bf16_round(((2.0 * u - 1.0) * scale).astype(np.float32))
    return out.reshape(rows, cols)


def prompt_tokens(seed: int, rid: int, n: int, vocab: int) -> np.ndarray:
    s = (seed + 1000003 * rid) & MASK64
    return (splitmix_at(s, np.arange(n, dtype=np.uint64)) % np.uint64(vocab)).astype(np.int64)


# ---------------------------------------------------------------- model
@dataclass
class Desc:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    tied_embeddings: bool = False
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    seed: int = 1


TINY = Desc(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn_dim=768, vocab=4096)
LLAMA_1B = Desc(n_layers=16, d_model=2048, n_heads=32, n_kv_heads=8, head_dim=64, ffn_dim=8192, vocab=128256,
                tied_embeddings=True)
LLAMA_8B = Desc(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336, vocab=128256)


class OracleModel:
    """fp32 Llama-style decoder over bf16-valued weights, paged KV cache.

    emulate_bf16=False is THE reference: everything in fp32.  emulate_bf16=True
    additionally rounds exactly where the CUDA path stores 16-bit values, so
    the remaining difference is accumulation order only: to bf16 for the GEMM
    inputs (RMSNorm outputs -- in decode the norm is folded into the GEMM, so
    the rounded tensor is the residual x itself --, attention output, SwiGLU
    output), to fp16 for the attention operands (roped q/k and v -- the KV
    cache -- and the softmax numerators fed to the P.V tensor-core product).
    """

    def __init__(self, desc: Desc, page_tokens: int = 16, emulate_bf16: bool = False, share_weights_with=None):
        self.d = desc
        self.B = page_tokens
        self.emul = emulate_bf16
        self._phase = "prefill"
        D, H, Hk, hd, F, V, L = (desc.d_model, desc.n_heads, desc.n_kv_heads, desc.head_dim, desc.ffn_dim,
                                 desc.vocab, desc.n_layers)
        s = desc.seed
        self.pages: Dict[int, np.ndarray] = {}
        half = hd // 2
        self.inv_freq = (1.0 / (desc.rope_theta ** (np.arange(half, dtype=np.float64) * 2.0 / hd))).astype(np.float32)
        # RMSNorm gains (bf16 values; the generator makes them 1, tests may set others):
        # per layer g_attn / g_mlp [d], and g_final [d]
        self.gains = dict(attn=[np.ones(D, np.float32) for _ in range(L)], mlp=[np.ones(D, np.float32) for _ in range(L)],
                          final=np.ones(D, np.float32))
        if share_weights_with is not None:  # same weights and gains, separate KV store
            o = share_weights_with
            self.emb, self.layers, self.lm, self.gains = o.emb, o.layers, o.lm, o.gains
            return
        self.emb = tensor_values(s, 0, V, D, D)
        self.layers = []
        for l in range(L):
            b = 1 + 7 * l
            self.layers.append(dict(
                wq=tensor_values(s, b + 0, H * hd, D, D),
                wk=tensor_values(s, b + 1, Hk * hd, D, D),
                wv=tensor_values(s, b + 2, Hk * hd, D, D),
                wo=tensor_values(s, b + 3, D, H * hd, H * hd),
                wg=tensor_values(s, b + 4, F, D, D),
                wu=tensor_values(s, b + 5, F, D, D),
                wd=tensor_values(s, b + 6, D, F, F),
            ))
        self.lm = self.emb if desc.tied_embeddings else tensor_values(s, 1 + 7 * L, V, D, D)

    # -- pieces
    def _r(self, x: np.ndarray) -> np.ndarray:
        return bf16_round(x) if self.emul else x

    def _r16(self, x: np.ndarray) -> np.ndarray:
        return f16_round(x) if self.emul else x

    def _norm_in(self, x: np.ndarray, g: np.ndarray) -> np.ndarray:
        """RMSNorm with gain g feeding a GEMM.  Emulation mirrors where the
        kernels round: prefill rounds the normalised rows; decode folds the norm
        into the GEMM (B operand = bf16(x * g), epilogue scales by 1/rms)."""
        if self.emul and self._phase == "decode":
            inv = 1.0 / np.sqrt(np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True) + np.float32(self.d.norm_eps))
            return (bf16_round(x * g) * inv).astype(np.float32)
        return self._r(self.rmsnorm(x, g))

    def rmsnorm(self, x: np.ndarray, g: Optional[np.ndarray] = None) -> np.ndarray:
        ms = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True)
        y = (x / np.sqrt(ms + np.float32(self.d.norm_eps))).astype(np.float32)
        return y if g is None else (y * g).astype(np.float32)

    def rope(self, x: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """x [T, heads, hd]; rotate-half convention, angle = pos * inv_freq (fp32)."""
        half = self.d.head_dim // 2
        ang = pos.astype(np.float32)[:, None] * self.inv_freq[None, :]
        c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
        a, b = x[..., :half], x[..., half:]
        return np.concatenate([a * c - b * s, b * c + a * s], axis=-1).astype(np.float32)

    def _page(self, pid: int) -> np.ndarray:
        p = self.pages.get(pid)
        if p is None:
            p = np.zeros((self.d.n_layers, 2, self.d.n_kv_heads, self.B, self.d.head_dim), dtype=np.float32)
            self.pages[pid] = p
        return p

    def _write_kv(self, l: int, row: Sequence[int], pos: np.ndarray, k: np.ndarray, v: np.ndarray):
        for t, p in enumerate(pos):
            pg = self._page(row[p // self.B])
            pg[l, 0, :, p % self.B, :] = k[t]
            pg[l, 1, :, p % self.B, :] = v[t]

    def _read_kv(self, l: int, row: Sequence[int], n: int):
        n_pages = (n + self.B - 1) // self.B
        ks = np.concatenate([self.pages[row[i]][l, 0] for i in range(n_pages)], axis=1)[:, :n]
        vs = np.concatenate([self.pages[row[i]][l, 1] for i in range(n_pages)], axis=1)[:, :n]
        return ks, vs  # [Hk, n, hd]

    def _attend(self, q: np.ndarray, ks: np.ndarray, vs: np.ndarray, qpos: np.ndarray) -> np.ndarray:
        """q [T, H, hd] at absolute positions qpos; causal over ks/vs [Hk, n, hd]."""
        H, Hk, hd = self.d.n_heads, self.d.n_kv_heads, self.d.head_dim
        g = H // Hk
        out = np.empty_like(q)
        n = ks.shape[1]
        mask = np.arange(n)[None, :] > qpos[:, None]  # [T, n]
        scale = np.float32(1.0 / math.sqrt(hd))
        for h in range(H):
            kh, vh = ks[h // g], vs[h // g]
            sc = (q[:, h, :] @ kh.T) * scale
            sc = np.where(mask, -np.inf, sc)
            sc = sc - sc.max(axis=1, keepdims=True)
            p = np.exp(sc)
            l = p.sum(axis=1, keepdims=True)
            if self.emul:  # the attention kernels feed fp16 P to the P.V tensor-core product
                p = f16_round(p)
            out[:, h, :] = (p @ vh) / l
        return out

    def _block(self, l: int, x: np.ndarray, rows: List[Sequence[int]], spans: List[np.ndarray]) -> np.ndarray:
        """One decoder layer over the concatenation of per-request token spans."""
        W = self.layers[l]
        H, Hk, hd = self.d.n_heads, self.d.n_kv_heads, self.d.head_dim
        h = self._norm_in(x, self.gains["attn"][l])
        q = (h @ W["wq"].T).reshape(-1, H, hd)
        k = (h @ W["wk"].T).reshape(-1, Hk, hd)
        v = self._r16((h @ W["wv"].T).reshape(-1, Hk, hd))
        pos_all = np.concatenate(spans)
        q, k = self._r16(self.rope(q, pos_all)), self._r16(self.rope(k, pos_all))
        o = np.empty_like(q)
        off = 0
        for row, pos in zip(rows, spans):
            t = len(pos)
            self._write_kv(l, row, pos, k[off:off + t], v[off:off + t])
            ks, vs = self._read_kv(l, row, int(pos[-1]) + 1)
            o[off:off + t] = self._attend(q[off:off + t], ks, vs, pos)
            off += t
        x = x + self._r(o.reshape(len(x), -1)) @ W["wo"].T
        h = self._norm_in(x, self.gains["mlp"][l])
        gate = h @ W["wg"].T
        a = self._r((gate / (1.0 + np.exp(-gate))) * (h @ W["wu"].T))
        return (x + a.astype(np.float32) @ W["wd"].T).astype(np.float32)

    def forward(self, tokens: np.ndarray, rows: List[Sequence[int]], spans: List[np.ndarray],
                want: Optional[np.ndarray] = None) -> np.ndarray:
        """Run all layers; return fp32 logits at the rows `want` (default: last of each span)."""
        x = self.emb[tokens].astype(np.float32)
        for l in range(self.d.n_layers):
            x = self._block(l, x, rows, spans)
        if want is None:
            want = np.cumsum([len(s) for s in spans]) - 1
        return (self._norm_in(x[want], self.gains["final"]) @ self.lm.T).astype(np.float32)

    # -- phase entry points (same semantics as sw_prefill_enqueue / sw_decode_enqueue)
    def prefill(self, prompts: List[np.ndarray], page_rows: List[Sequence[int]]) -> np.ndarray:
        toks = np.concatenate(prompts)
        spans = [np.arange(len(p)) for p in prompts]
        self._phase = "prefill"
        return self.forward(toks, page_rows, spans)

    def decode(self, tokens: Sequence[int], positions: Sequence[int], page_rows: List[Sequence[int]]) -> np.ndarray:
        spans = [np.array([p]) for p in positions]
        self._phase = "decode"
        return self.forward(np.asarray(tokens, dtype=np.int64), page_rows, spans)

    def release(self, page_row: Sequence[int]):
        for p in page_row:
            self.pages.pop(p, None)


def argmax_first(logits: np.ndarray) -> np.ndarray:
    return np.argmax(logits, axis=-1)


def top2_margin(logits: np.ndarray) -> np.ndarray:
    part = np.partition(logits, -2, axis=-1)
    return part[..., -1] - part[..., -2]


def generate_greedy(model: OracleModel, prompt: np.ndarray, n_out: int, page_row: Sequence[int]):
    """Serial reference for one request: x_1 from the prompt, then n_out-1 more steps.

    Returns (tokens x_1..x_out, per-step fp32 logits)."""
    logits = [model.prefill([prompt], [page_row])[0]]
    toks = [int(argmax_first(logits[-1]))]
    for g in range(1, n_out):
        lg = model.decode([toks[-1]], [len(prompt) + g - 1], [page_row])[0]
        logits.append(lg)
        toks.append(int(argmax_first(lg)))
    return toks, logits

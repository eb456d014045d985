"""Python handle over the C-ABI model/arena objects (tests and bench only).

Device memory for optional logits comes from PyTorch (plumbing); every
computation happens inside libsplitwise.so.
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import Batch, ModelDesc, RunResult, check, lib, parse_run_text, spec_string, _take_text


def _i32(xs) -> ctypes.Array:
    arr = (ctypes.c_int32 * len(xs))(*[int(x) for x in xs])
    return arr


def model_desc(d, max_prefill_tokens: int, max_decode_batch: int) -> ModelDesc:
    return ModelDesc(n_layers=d.n_layers, d_model=d.d_model, n_heads=d.n_heads, n_kv_heads=d.n_kv_heads,
                     head_dim=d.head_dim, ffn_dim=d.ffn_dim, vocab=d.vocab,
                     tied_embeddings=1 if d.tied_embeddings else 0, rope_theta=d.rope_theta, norm_eps=d.norm_eps,
                     seed=d.seed, max_prefill_tokens=max_prefill_tokens, max_decode_batch=max_decode_batch)


class Engine:
    """One model (weights generated on the device) + one paged KV arena."""

    def __init__(self, desc, max_prefill_tokens=4096, max_decode_batch=64, n_pages=4096, n_slots=64,
                 max_pages_per_slot=64, max_out=64, device=0, kv_reserve_bytes=2 << 30, max_pages=None):
        """n_pages=None sizes the KV arena from the device's free HBM after the
        weights are resident (sw_kv_capacity_pages: the reference's
        derive_kv_capacity with budget = free - kv_reserve_bytes), capped at
        max_pages when given."""
        self.desc = desc
        L = lib()
        self.model = ctypes.c_void_p()
        md = model_desc(desc, max_prefill_tokens, max_decode_batch)
        check(L.sw_model_create(ctypes.byref(md), device, ctypes.byref(self.model)))
        if n_pages is None:
            cap = ctypes.c_int64()
            check(L.sw_kv_capacity_pages(ctypes.byref(md), device, int(kv_reserve_bytes), ctypes.byref(cap)))
            n_pages = int(cap.value) if max_pages is None else min(int(cap.value), int(max_pages))
        self.kv = ctypes.c_void_p()
        check(L.sw_kv_arena_create(self.model, n_pages, n_slots, max_pages_per_slot, max_out, ctypes.byref(self.kv)))
        self.n_pages, self.n_slots, self.max_pages, self.max_out = n_pages, n_slots, max_pages_per_slot, max_out

    def close(self):
        L = lib()
        if self.kv:
            check(L.sw_kv_arena_destroy(self.kv))
            self.kv = ctypes.c_void_p()
        if self.model:
            check(L.sw_model_destroy(self.model))
            self.model = ctypes.c_void_p()

    # -- kernel level
    def _stream(self):
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def prefill(self, slots: Sequence[int], prompts: Sequence[np.ndarray], page_rows: Sequence[Sequence[int]],
                out_index: Optional[Sequence[int]] = None, logits: bool = True,
                positions: Optional[Sequence[int]] = None):
        """Prefill prompts (or prompt chunks: `positions` = each chunk's first position, a multiple of
        128, with the earlier positions already in the slot's pages; page_rows then cover [0, pos + len))."""
        import torch

        n = len(slots)
        out = torch.empty((n, self.desc.vocab), dtype=torch.float32, device="cuda") if logits else None
        toks = np.concatenate([np.asarray(p, dtype=np.int64) for p in prompts])
        keep = [_i32(slots), _i32([len(p) for p in prompts]), _i32(toks), _i32([x for r in page_rows for x in r]),
                _i32(out_index if out_index is not None else [0] * n),
                _i32(positions) if positions is not None else None]
        b = Batch(n=n, slots=keep[0], n_tokens=keep[1], tokens=keep[2], page_rows=keep[3], out_index=keep[4],
                  logits_out=out.data_ptr() if out is not None else None)
        if keep[5] is not None:
            b.positions = keep[5]
        check(lib().sw_prefill_enqueue(self.model, self.kv, ctypes.byref(b), self._stream()))
        torch.cuda.synchronize()
        return out.cpu().numpy() if out is not None else None

    def decode(self, slots, positions, tokens=None, new_page=None, out_index=None, logits: bool = True):
        import torch

        n = len(slots)
        out = torch.empty((n, self.desc.vocab), dtype=torch.float32, device="cuda") if logits else None
        keep = [_i32(slots), _i32(positions), _i32(tokens) if tokens is not None else None,
                _i32(new_page) if new_page is not None else None,
                _i32(out_index) if out_index is not None else None]
        b = Batch(n=n, slots=keep[0], positions=keep[1], logits_out=out.data_ptr() if out is not None else None)
        if keep[2] is not None:
            b.tokens = keep[2]
        if keep[3] is not None:
            b.new_page = keep[3]
        if keep[4] is not None:
            b.out_index = keep[4]
        check(lib().sw_decode_enqueue(self.model, self.kv, ctypes.byref(b), self._stream()))
        torch.cuda.synchronize()
        return out.cpu().numpy() if out is not None else None

    def mixed(self, slots: Sequence[int], prompts: Sequence[np.ndarray], page_rows: Sequence[Sequence[int]],
              dec_slots, dec_positions, dec_tokens=None, dec_new_page=None, out_index=None, dec_out_index=None,
              logits: bool = True):
        """One fused mixed step (sw_mixed_enqueue): prompts and decode rows in one
        pass.  Returns logits [prompts + decode rows, vocab] (prompts first)."""
        import torch

        n, nd = len(slots), len(dec_slots)
        out = torch.empty((n + nd, self.desc.vocab), dtype=torch.float32, device="cuda") if logits else None
        toks = np.concatenate([np.asarray(p, dtype=np.int64) for p in prompts])
        keep = [_i32(slots), _i32([len(p) for p in prompts]), _i32(toks), _i32([x for r in page_rows for x in r]),
                _i32(out_index if out_index is not None else [0] * n), _i32(dec_slots), _i32(dec_positions)]
        pb = Batch(n=n, slots=keep[0], n_tokens=keep[1], tokens=keep[2], page_rows=keep[3], out_index=keep[4],
                   logits_out=out.data_ptr() if out is not None else None)
        db = Batch(n=nd, slots=keep[5], positions=keep[6])
        for field, vals in (("tokens", dec_tokens), ("new_page", dec_new_page), ("out_index", dec_out_index)):
            if vals is not None:
                keep.append(_i32(vals))
                setattr(db, field, keep[-1])
        check(lib().sw_mixed_enqueue(self.model, self.kv, ctypes.byref(pb), ctypes.byref(db), self._stream()))
        torch.cuda.synchronize()
        return out.cpu().numpy() if out is not None else None

    def tensor(self, name: str):
        """(device pointer, numel) of a weight tensor."""
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        check(lib().sw_model_tensor(self.model, name.encode(), ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def tensor_numpy(self, name: str) -> np.ndarray:
        """Copy a bf16 weight tensor to the host as float32 values."""
        import torch

        ptr, n = self.tensor(name)
        host = device_view(ptr, (n,), "<i2").cpu().numpy().view(np.uint16)
        return (host.astype(np.uint32) << 16).view(np.float32)

    def write_tensor(self, name: str, values: np.ndarray):
        """Overwrite a bf16 weight tensor (e.g. RMSNorm gains) with `values`,
        rounded to nearest-even bf16; returns the stored values as float32."""
        import torch

        ptr, n = self.tensor(name)
        v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        if v.size != n:
            raise ValueError(f"{name}: {v.size} values for {n} elements")
        t = torch.from_numpy(v).to(torch.bfloat16)
        device_view(ptr, (n,), "<i2").copy_(t.view(torch.int16).cuda())
        torch.cuda.synchronize()
        return t.float().numpy()

    def weight_checksum(self) -> int:
        v = ctypes.c_uint64()
        check(lib().sw_model_weight_checksum(self.model, ctypes.byref(v)))
        return v.value

    # -- run level
    def run(self, spec) -> RunResult:
        s = spec if isinstance(spec, str) else spec_string(spec)
        out = ctypes.c_void_p()
        check(lib().sw_engine_run(self.model, self.kv, s.encode(), ctypes.byref(out)))
        res = parse_run_text(_take_text(out))
        return res

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class _DevArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def device_view(ptr: int, shape, typestr: str):
    """Zero-copy torch view of device memory owned by the library."""
    import torch

    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda")


def parse_devpages(res: RunResult) -> Dict[int, List[int]]:
    out = {}
    for line in res.text.splitlines():
        if line.startswith("#devpages "):
            rid, _, row = line[10:].partition(":")
            out[int(rid)] = [int(x) for x in row.split("|") if x]
    return out

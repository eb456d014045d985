"""B200-native split-phase (prefill || decode) inference engine.

The product is the in-tree shared library ``libsplitwise.so`` (C++20 host engine
+ hand-written sm_100a CUDA kernels) behind the C-ABI declared in
``include/splitwise.h``.  This module is a thin ctypes binding used by the
tests and ``bench.py``; it performs no computation itself.  There is no CPU or
PyTorch fallback: if the library is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsplitwise.so")

SW_OK, SW_ECONFIG, SW_EIO, SW_ECONTRACT, SW_ECUDA = 0, -2, -3, -4, -5


class SplitwiseError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(SplitwiseError):
    pass


class IoError(SplitwiseError):
    pass


class ContractViolation(SplitwiseError):
    pass


class CudaError(SplitwiseError):
    pass


_ERRORS = {SW_ECONFIG: ConfigError, SW_EIO: IoError, SW_ECONTRACT: ContractViolation, SW_ECUDA: CudaError}

_lib: Optional[ctypes.CDLL] = None


class ModelDesc(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int32),
        ("d_model", ctypes.c_int32),
        ("n_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("ffn_dim", ctypes.c_int32),
        ("vocab", ctypes.c_int32),
        ("tied_embeddings", ctypes.c_int32),
        ("rope_theta", ctypes.c_float),
        ("norm_eps", ctypes.c_float),
        ("seed", ctypes.c_uint64),
        ("max_prefill_tokens", ctypes.c_int32),
        ("max_decode_batch", ctypes.c_int32),
    ]


class Batch(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("slots", ctypes.POINTER(ctypes.c_int32)),
        ("n_tokens", ctypes.POINTER(ctypes.c_int32)),
        ("positions", ctypes.POINTER(ctypes.c_int32)),
        ("tokens", ctypes.POINTER(ctypes.c_int32)),
        ("page_rows", ctypes.POINTER(ctypes.c_int32)),
        ("new_page", ctypes.POINTER(ctypes.c_int32)),
        ("out_index", ctypes.POINTER(ctypes.c_int32)),
        ("logits_out", ctypes.c_void_p),
    ]


def lib() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C paper_2505_03763_b200/csrc)")
        L = ctypes.CDLL(LIB_PATH)
        c_int, c_char_p, c_void_p = ctypes.c_int, ctypes.c_char_p, ctypes.c_void_p
        L.sw_last_error.restype = c_char_p
        L.sw_free.argtypes = [c_void_p]
        L.sw_sim_run.argtypes = [c_char_p, ctypes.POINTER(c_void_p)]
        L.sw_sim_run.restype = c_int
        L.sw_launch_count.restype = ctypes.c_ulonglong
        L.sw_transfer_bytes.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)] * 2
        L.sw_transfer_bytes.restype = None
        for name, args in {
            "sw_engine_run": [c_void_p, c_void_p, c_char_p, ctypes.POINTER(c_void_p)],
            "sw_replay": [c_char_p, ctypes.POINTER(c_void_p)],
            "sw_model_create": [ctypes.POINTER(ModelDesc), c_int, ctypes.POINTER(c_void_p)],
            "sw_model_destroy": [c_void_p],
            "sw_model_weight_checksum": [c_void_p, ctypes.POINTER(ctypes.c_uint64)],
            "sw_model_tensor": [c_void_p, c_char_p, ctypes.POINTER(c_void_p), ctypes.POINTER(ctypes.c_int64)],
            "sw_kv_arena_create": [c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.POINTER(c_void_p)],
            "sw_kv_arena_destroy": [c_void_p],
            "sw_kv_capacity_pages": [ctypes.POINTER(ModelDesc), c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
            "sw_kv_arena_views": [c_void_p] + [ctypes.POINTER(c_void_p)] * 4,
            "sw_sm_partition": [c_int, c_int, ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p),
                                ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
            "sw_prefill_enqueue": [c_void_p, c_void_p, ctypes.POINTER(Batch), c_void_p],
            "sw_decode_enqueue": [c_void_p, c_void_p, ctypes.POINTER(Batch), c_void_p],
            "sw_mixed_enqueue": [c_void_p, c_void_p, ctypes.POINTER(Batch), ctypes.POINTER(Batch), c_void_p],
            "sw_op_gemm": [c_void_p, c_void_p, c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                           ctypes.c_int32, c_void_p],
            "sw_op_rmsnorm": [c_void_p, c_void_p, c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_float,
                              c_void_p],
        }.items():
            if not hasattr(L, name):
                continue  # reported by tests/test_capi.py::test_exports
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c_int
        _lib = L
    return _lib


EXPORTED_SYMBOLS = [
    "sw_last_error", "sw_free", "sw_launch_count", "sw_transfer_bytes", "sw_sim_run", "sw_engine_run", "sw_replay", "sw_model_create", "sw_model_destroy",
    "sw_model_weight_checksum", "sw_model_tensor", "sw_kv_arena_create", "sw_kv_arena_destroy", "sw_kv_capacity_pages",
    "sw_kv_arena_views", "sw_sm_partition", "sw_prefill_enqueue", "sw_decode_enqueue", "sw_mixed_enqueue", "sw_op_gemm", "sw_op_rmsnorm",
]


def check(code: int) -> None:
    if code != SW_OK:
        msg = lib().sw_last_error().decode(errors="replace")
        raise _ERRORS.get(code, SplitwiseError)(code, msg)


def _take_text(ptr: ctypes.c_void_p) -> str:
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().sw_free(ptr)


def spec_string(spec: Dict[str, object]) -> str:
    return ";".join(f"{k}={v}" for k, v in spec.items())


@dataclass
class RunResult:
    """Parsed output of sw_sim_run / sw_engine_run."""
    text: str
    event_log: str = ""
    report: Dict[str, float] = field(default_factory=dict)
    requests: List[Dict[str, float]] = field(default_factory=list)
    pages: Dict[int, List[int]] = field(default_factory=dict)
    journal: List[tuple] = field(default_factory=list)
    tokens: Dict[int, List[int]] = field(default_factory=dict)
    extra: Dict[str, str] = field(default_factory=dict)


def _kv_line(line: str) -> Dict[str, str]:
    out = {}
    for item in line.split(";"):
        if item:
            k, _, v = item.partition("=")
            out[k] = v
    return out


def parse_run_text(text: str) -> RunResult:
    res = RunResult(text=text)
    log_lines = []
    for line in text.splitlines():
        if line.startswith("#report "):
            res.report = {k: float(v) for k, v in _kv_line(line[8:]).items()}
        elif line.startswith("#request "):
            res.requests.append({k: float(v) for k, v in _kv_line(line[9:]).items()})
        elif line.startswith("#pages "):
            rid, _, row = line[7:].partition(":")
            res.pages[int(rid)] = [int(x) for x in row.split("|") if x]
        elif line.startswith("#journal"):
            body = line[8:].strip()
            res.journal = [tuple(int(x) for x in e.split(":")) for e in body.split("|") if e]
        elif line.startswith("#tokens "):
            rid, _, row = line[8:].partition(":")
            res.tokens[int(rid)] = [int(x) for x in row.split("|") if x]
        elif line.startswith("#"):
            key, _, val = line[1:].partition(" ")
            res.extra[key] = val
        else:
            log_lines.append(line)
    res.event_log = "\n".join(log_lines) + "\n"
    return res


def sim_run(spec) -> RunResult:
    """Virtual-clock run of a policy (parity backend for the scheduler API)."""
    s = spec if isinstance(spec, str) else spec_string(spec)
    out = ctypes.c_void_p()
    check(lib().sw_sim_run(s.encode(), ctypes.byref(out)))
    return parse_run_text(_take_text(out))


def replay(events_path: str) -> RunResult:
    """Rebuild the report of a written events.csv (writes replay_report.json next to it)."""
    out = ctypes.c_void_p()
    check(lib().sw_replay(str(events_path).encode(), ctypes.byref(out)))
    return parse_run_text(_take_text(out))


def launch_count() -> int:
    return int(lib().sw_launch_count())


def transfer_bytes():
    h, d = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    lib().sw_transfer_bytes(ctypes.byref(h), ctypes.byref(d))
    return int(h.value), int(d.value)

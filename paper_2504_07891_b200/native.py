"""ctypes binding of ``libspecreason_b200.so`` (the C-ABI in
``include/specreason_b200.h``).  The library is built in-tree by
``__graft_entry__.build()`` (``csrc/Makefile``); importing this module on a
machine without it raises -- there is no fallback path."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).with_name("libspecreason_b200.so")

SR_PAGE = 64
SR_HEAD_DIM = 128


class ModelDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn",
        "vocab_rows", "vocab_text")] + [("rms_eps", C.c_float)] + [
        (n, C.c_int32) for n in ("max_pos", "max_tokens", "max_new", "n_pages", "tp_world",
                                 "tp_rank", "vocab_base")]


class LayerPtrs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wd")]


class ModelPtrs(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("ln_f", C.c_void_p), ("lm_head", C.c_void_p),
                ("layers", C.POINTER(LayerPtrs)), ("rope", C.c_void_p),
                ("k_pool", C.c_void_p), ("v_pool", C.c_void_p), ("workspace", C.c_void_p)]


class Readout(C.Structure):
    _fields_ = [("score", C.c_int32), ("accept", C.c_int32), ("margin", C.c_float),
                ("argmax", C.c_int32)]


class Timing(C.Structure):
    _fields_ = [("prefill_ms", C.c_float), ("decode_ms", C.c_float),
                ("prefill_tokens", C.c_int32), ("decode_tokens", C.c_int32)]


EXPORTS = {
    "sr_abi_version": (C.c_int, []),
    "sr_last_error": (C.c_char_p, []),
    "sr_workspace_bytes": (C.c_size_t, [C.POINTER(ModelDesc)]),
    "sr_model_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(ModelPtrs), C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
    "sr_model_destroy": (C.c_int, [C.c_void_p]),
    "sr_generate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                              C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sr_score": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                           C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "sr_forward_logits": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_int32, C.c_void_p, C.c_void_p]),
    "sr_last_timing": (C.c_int, [C.c_void_p, C.POINTER(Timing)]),
    "sr_verify_tokens": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "sr_score_batch": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                 C.c_void_p]),
    "sr_step_batch": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sr_debug_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "sr_debug_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "sr_tp_unique_id": (C.c_int, [C.c_void_p]),
    "sr_tp_comm_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "sr_tp_comm_destroy": (C.c_int, [C.c_void_p]),
    "sr_model_set_tp": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sr_tp_peer_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "sr_tp_peer_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sr_tp_peer_open": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sr_tp_peer_base": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "sr_tp_peer_attach": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sr_tp_peer_destroy": (C.c_int, [C.c_void_p]),
    "sr_model_set_tp_peer": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sr_model_set_decode_tiles": (C.c_int, [C.c_void_p, C.c_void_p]),
}

_lib = None


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str) -> None:
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def load() -> C.CDLL:
    """Load (once) and type the library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SR_LIB", LIB_PATH))
    if not path.exists():
        raise FileNotFoundError(
            f"{path} is missing: run __graft_entry__.build() (make -C paper_2504_07891_b200/csrc)")
    lib = C.CDLL(str(path))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(fn: str, rc: int) -> None:
    if rc != 0:
        msg = load().sr_last_error().decode(errors="replace")
        raise NativeError(fn, rc, msg)

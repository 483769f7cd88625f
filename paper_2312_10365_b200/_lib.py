"""ctypes loader for libspt_ffn.so (the C ABI declared in include/spt_ffn.h).

Loading fails loudly if the shared library is missing: there is no fallback
implementation of any kind behind this package.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspt_ffn.so")

SPT_OK, SPT_ERR_INVALID_ARGUMENT, SPT_ERR_UNSUPPORTED, SPT_ERR_WORKSPACE_TOO_SMALL, SPT_ERR_CUDA = range(5)
SPT_F32, SPT_BF16 = 0, 1
SPT_ACT_RELU, SPT_ACT_GELU, SPT_ACT_SWIGLU = 0, 1, 2
SPT_GATE_SIGMOID, SPT_GATE_NONE = 0, 1
SPT_ROUTE_LOGITS_IN = 1
SPT_BWD_ACCUMULATE_DW = 1
SPT_FFN_DETERMINISTIC = 1
SPT_TILE_M = 128

# every symbol include/spt_ffn.h declares
EXPORTED = ("spt_ffn_sizes", "spt_ffn_route", "spt_ffn_forward", "spt_ffn_backward",
            "spt_ffn_balance_loss", "spt_status_string", "spt_ffn_abi_version", "spt_ffn_launch_count",
            "spt_ffn_profile_enable", "spt_ffn_profile_read",
            "spt_ffn_lora_sizes", "spt_ffn_lora_forward", "spt_ffn_lora_backward",  # ABI 3
            "spt_mha_topl")  # ABI 4


class spt_ffn_desc(ctypes.Structure):
    _fields_ = [("n_tokens", ctypes.c_int64), ("d_model", ctypes.c_int32), ("d_ff", ctypes.c_int32),
                ("n_blocks", ctypes.c_int32), ("top_k", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("act", ctypes.c_int32), ("gate", ctypes.c_int32),
                ("balance_weight", ctypes.c_float),  # ABI 2
                ("flags", ctypes.c_uint32)]  # ABI 5: SPT_FFN_DETERMINISTIC


class spt_route_buf(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("logits", "topk_idx", "topk_gate", "block_offsets",
                                               "bucket_token", "bucket_gate", "pair_slot",
                                               "tile_offsets")]


class spt_lora(ctypes.Structure):  # ABI 3: LoRA factors (device pointers)
    _fields_ = [("rank", ctypes.c_int32)] + [(n, ctypes.c_void_p) for n in ("b1", "c1", "b2", "c2")]


class spt_lora_grads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("db1", "dc1", "db2", "dc2")]


class spt_topl_desc(ctypes.Structure):  # ABI 4: sparse-MHA top-L selection
    _fields_ = [(n, ctypes.c_int32) for n in ("n_heads", "n_q", "n_k", "n_codebooks",
                                              "n_codewords", "top_l", "causal")]


class SptError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {status_string(code)} ({code})")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libspt_ffn.so not built ({LIB_PATH}); run `make` or "
                              "__graft_entry__.build() -- there is no fallback path")
        L = ctypes.CDLL(LIB_PATH)
        P, D, R = ctypes.c_void_p, ctypes.POINTER(spt_ffn_desc), ctypes.POINTER(spt_route_buf)
        sz = ctypes.POINTER(ctypes.c_size_t)
        L.spt_ffn_sizes.argtypes = [D, sz, sz]
        L.spt_ffn_route.argtypes = [D, P, P, ctypes.c_uint, R, P, ctypes.c_size_t, P]
        L.spt_ffn_forward.argtypes = [D, P, P, P, R, P, P, P, ctypes.c_size_t, P]
        L.spt_ffn_backward.argtypes = [D, P, P, P, P, R, P, P, P, P, P, P, P, ctypes.c_uint, P,
                                       ctypes.c_size_t, P, P]
        L.spt_ffn_balance_loss.argtypes = [D, R, P, P, ctypes.c_size_t, P]
        LO, LG = ctypes.POINTER(spt_lora), ctypes.POINTER(spt_lora_grads)
        L.spt_ffn_lora_sizes.argtypes = [D, ctypes.c_int32, sz, sz]
        L.spt_ffn_lora_forward.argtypes = [D, P, P, P, LO, R, P, P, P, ctypes.c_size_t, P]
        L.spt_ffn_lora_backward.argtypes = [D, P, P, P, P, LO, R, P, P, P, LG, P, P, ctypes.c_uint,
                                            P, ctypes.c_size_t, P, P]
        L.spt_mha_topl.argtypes = [ctypes.POINTER(spt_topl_desc), P, P, P, P]
        for f in ("spt_ffn_sizes", "spt_ffn_route", "spt_ffn_forward", "spt_ffn_backward",
                  "spt_ffn_balance_loss", "spt_ffn_lora_sizes", "spt_ffn_lora_forward",
                  "spt_ffn_lora_backward", "spt_mha_topl"):
            getattr(L, f).restype = ctypes.c_int
        L.spt_status_string.argtypes = [ctypes.c_int]
        L.spt_status_string.restype = ctypes.c_char_p
        L.spt_ffn_abi_version.restype = ctypes.c_int
        L.spt_ffn_launch_count.restype = ctypes.c_uint64
        L.spt_ffn_profile_enable.argtypes = [ctypes.c_int]
        L.spt_ffn_profile_enable.restype = ctypes.c_int
        L.spt_ffn_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        L.spt_ffn_profile_read.restype = ctypes.c_int64
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().spt_status_string(code).decode()


def check(fn: str, code: int) -> None:
    if code != SPT_OK:
        raise SptError(fn, code)

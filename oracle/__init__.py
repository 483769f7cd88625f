"""CPU fp64 oracle of SPT's routed FFN (arXiv 2312.10365) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2312_10365_b200``) never imports it, and it never imports the product.

Two formulations live here:
  * ``spt_oracle.c`` (loaded through ctypes): O2, the per-token form
    y_t = sum_{b in S_t} g * act(x_t W1_b^T) W2_b, plus the backward, top-k and
    bucketing -- see the C file's header for passages and readings.
  * ``alg4_forward`` below: O3, Algorithm 4 written literally
    as a loop over blocks with token masks, using numpy matmul as the GEMM step
    and accumulation for line 5 (reading c1).
Everything is fp64.  Parity status: pinned (tests/test_oracle_*.py); no
function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spt_oracle.c")
_LIB = os.path.join(_HERE, "libspt_oracle.so")

ACT_RELU, ACT_GELU, ACT_SWIGLU = 0, 1, 2
GATE_SIGMOID, GATE_NONE = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, i32, P = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        _lib.spt_oracle_router.argtypes = [i64, i32, i32, P, P, P]
        _lib.spt_oracle_topk.argtypes = [i64, i32, i32, P, P]
        _lib.spt_oracle_bucket.argtypes = [i64, i32, i32, P, i32, P, P, P, P]
        _lib.spt_oracle_forward.argtypes = [i64, i32, i32, i32, i32, i32, i32, P, P, P, P, P, P, i64, P]
        _lib.spt_oracle_backward_tokens.argtypes = [i64, i32, i32, i32, i32, i32, i32,
                                                    P, P, P, P, P, P, P, P, i64, P, P]
        _lib.spt_oracle_backward_blocks.argtypes = [i64, i32, i32, i32, i32, i32, i32,
                                                    P, P, P, P, P, P, P, i32, P, P, P]
        _lib.spt_oracle_forward_gemm_flops.argtypes = [i64, i32, i32, i32, i32, i32]
        _lib.spt_oracle_balance.argtypes = [i64, i32, i32, P, P, P]
        _lib.spt_oracle_balance.restype = ctypes.c_double
        _lib.spt_oracle_forward_gemm_flops.restype = ctypes.c_double
        _lib.spt_oracle_max_threads.restype = ctypes.c_int
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def max_threads() -> int:
    return int(lib().spt_oracle_max_threads())


def router(x, w_r) -> np.ndarray:
    """fp64 logits x_R = x W_R; w_r is W_R^T [G, d]."""
    x, w_r = _f64(x), _f64(w_r)
    T, d = x.shape
    G = w_r.shape[0]
    out = np.empty((T, G), np.float64)
    lib().spt_oracle_router(T, d, G, _ptr(x), _ptr(w_r), _ptr(out))
    return out


def topk(logits_f32, k) -> np.ndarray:
    """Top-k by |logit| bit pattern, ties -> lower id, ids ascending (c3, c4)."""
    lg = _f32(logits_f32)
    T, G = lg.shape
    out = np.empty((T, k), np.int32)
    if lib().spt_oracle_topk(T, G, k, _ptr(lg), _ptr(out)) != 0:
        raise ValueError("top-k: need 1 <= k <= G (SPEC S:325)")
    return out


def bucket(topk_idx, G, tile_m=128) -> dict:
    """Block-major bucket layout of the (token, block) pairs (Alg. 4 lines 2-3)."""
    ti = np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, k = ti.shape
    bo = np.empty(G + 1, np.int32)
    bt = np.empty(T * k, np.int32)
    ps = np.empty(T * k, np.int32)
    to = np.empty(G + 1, np.int32)
    rc = lib().spt_oracle_bucket(T, G, k, _ptr(ti), tile_m, _ptr(bo), _ptr(bt), _ptr(ps), _ptr(to))
    if rc != 0:
        raise ValueError("inconsistent routing decision")
    return {"block_offsets": bo, "bucket_token": bt, "pair_slot": ps, "tile_offsets": to}


def forward(x, w1, w2, logits, topk_idx, act, gate, tokens=None) -> np.ndarray:
    """O2 forward.  Returns y [T, d] fp64 (rows outside ``tokens`` are NaN)."""
    x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
    lg, ti = _f64(logits), np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, d = x.shape
    D = w2.shape[0]
    G = lg.shape[1]
    k = ti.shape[1]
    y = np.full((T, d), np.nan)
    tk = None if tokens is None else np.ascontiguousarray(tokens, dtype=np.int64)
    lib().spt_oracle_forward(T, d, D, G, k, act, gate, _ptr(x), _ptr(w1), _ptr(w2), _ptr(lg),
                             _ptr(ti), _ptr(tk), 0 if tk is None else len(tk), _ptr(y))
    return y


def balance(logits, topk_idx, want_grad=True):
    """Load-balancing loss L = G sum_g f_g pbar_g and dL/dx_R [T, G]
    (reading c18: f_g = n_g / (T k)).  spt_oracle.c."""
    lg, ti = _f64(logits), np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, G = lg.shape
    k = ti.shape[1] if ti.ndim == 2 else 1
    dl = np.zeros((T, G)) if want_grad else None
    L = float(lib().spt_oracle_balance(T, G, k, _ptr(lg), _ptr(ti), _ptr(dl)))
    return L, dl


def backward(x, w1, w2, w_r, logits, topk_idx, dy, act, gate, tokens=None, blocks=None,
             want_tokens=True, want_blocks=True, lb_weight=0.0) -> dict:
    """O2 backward: dx, dgate (per token subset) and dw1, dw2, dw_r (per block subset).

    lb_weight = lambda > 0 adds the gradient of lambda * L_balance (balance()):
    x_R = x W_R gives dW_R += lambda * dL/dx_R^T X and dX += lambda * dL/dx_R W_R^T
    (every block, selected or not); dgate is the task loss's only."""
    x, w1, w2, w_r, dy = _f64(x), _f64(w1), _f64(w2), _f64(w_r), _f64(dy)
    lg, ti = _f64(logits), np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, d = x.shape
    D = w2.shape[0]
    G = lg.shape[1]
    k = ti.shape[1]
    mp = 2 if act == ACT_SWIGLU else 1
    out = {}
    # entries the oracle does not compute (a token / block subset) are NaN; a full
    # call writes every entry, so it skips the (single-threaded) NaN fill
    fill = np.full if tokens is not None else (lambda shape, v: np.empty(shape))
    if want_tokens:
        dx = fill((T, d), np.nan)
        dg = fill((T, k), np.nan)
        tk = None if tokens is None else np.ascontiguousarray(tokens, dtype=np.int64)
        lib().spt_oracle_backward_tokens(T, d, D, G, k, act, gate, _ptr(x), _ptr(w1), _ptr(w2),
                                         _ptr(w_r), _ptr(lg), _ptr(ti), _ptr(dy), _ptr(tk),
                                         0 if tk is None else len(tk), _ptr(dx), _ptr(dg))
        out["dx"], out["dgate"] = dx, dg
    if want_blocks:
        fill = np.full if blocks is not None else (lambda shape, v: np.empty(shape))
        dw1 = fill((mp, D, d) if mp == 2 else (D, d), np.nan)
        dw2 = fill((D, d), np.nan)
        dwr = fill((G, d), np.nan)
        bl = None if blocks is None else np.ascontiguousarray(blocks, dtype=np.int32)
        lib().spt_oracle_backward_blocks(T, d, D, G, k, act, gate, _ptr(x), _ptr(w1), _ptr(w2),
                                         _ptr(lg), _ptr(ti), _ptr(dy), _ptr(bl),
                                         0 if bl is None else len(bl), _ptr(dw1), _ptr(dw2),
                                         _ptr(dwr))
        out["dw1"], out["dw2"], out["dw_r"] = dw1, dw2, dwr
    if lb_weight:
        _, dl = balance(lg, ti)
        if want_tokens:
            rows = slice(None) if tokens is None else np.asarray(tokens)
            out["dx"][rows] += lb_weight * (dl[rows] @ w_r)
        if want_blocks:
            bl = slice(None) if blocks is None else np.asarray(blocks)
            out["dw_r"][bl] += lb_weight * (dl[:, bl].T @ x)
    return out


def forward_gemm_flops(T, d, D, G, k, act) -> float:
    return float(lib().spt_oracle_forward_gemm_flops(T, d, D, G, k, act))


# ----------------------------------------------------------------- O3 form
def _act_np(act, zg, zu=None):
    if act == ACT_RELU:
        return np.maximum(zg, 0.0)
    if act == ACT_GELU:
        from scipy.special import erf
        return 0.5 * zg * (1.0 + erf(zg / np.sqrt(2.0)))
    return zg / (1.0 + np.exp(-zg)) * zu


def alg4_forward(x, w1, w2, logits, topk_idx, act, gate) -> np.ndarray:
    """O3: Algorithm 4 "The procedure of BSpMV", literally:

      for block i = 1..G:                                   (line 1)
          Mask_T <- eq(Indices, i)                          (line 2)
          X_i    <- X[Mask_T]                               (line 3)
          H      <- act(X_i W_I[i])                         (line 4)
          Y[Mask_T] += gate * (H W_O[i])                    (line 5, reading c1/c2)
    """
    x = np.asarray(x, np.float64)
    w1 = np.asarray(w1, np.float64)
    w2 = np.asarray(w2, np.float64)
    lg = np.asarray(logits, np.float64)
    T, d = x.shape
    D = w2.shape[0]
    G = lg.shape[1]
    bw = D // G
    y = np.zeros((T, d))
    for i in range(G):
        mask_tok = (topk_idx == i).any(axis=1)              # eq(Indices, i)
        if not mask_tok.any():
            continue
        X_i = x[mask_tok]
        rows = slice(i * bw, (i + 1) * bw)
        if act == ACT_SWIGLU:
            H = _act_np(act, X_i @ w1[0, rows].T, X_i @ w1[1, rows].T)
        else:
            H = _act_np(act, X_i @ w1[rows].T)
        g = 1.0 / (1.0 + np.exp(-lg[mask_tok, i])) if gate == GATE_SIGMOID else np.ones(X_i.shape[0])
        y[mask_tok] += (g[:, None] * H) @ w2[rows]
    return y

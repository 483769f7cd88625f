"""fp64 oracle of the LoRA-wrapped routed FFN -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module; it never imports the product.

What it computes (the paper's fine-tuning mode):
  * LoRA (Eq. 5): a projection Y = XW becomes
        Y = XW + XBC,   W frozen, B in R^{d x r}, C in R^{r x h} trained.
  * SPT wraps both FFN projections in LoRA (the Model Adapter log,
    PAPER.md:1323-1328: "ffd.fc1 Linear -> LoRALinear", "ffd.fc2 ..."),
    rank r = d_lora (default 16), and then routes the FFN
    (§4.2): block b keeps the hidden units
    [b bw, (b+1) bw), i.e. the block's columns of W_I + B_I C_I and rows of
    W_O + B_O C_O (reading c5 applied to the LoRA-wrapped weights, DESIGN.md
    reading c19).
  * Per token t with activated blocks S_t (ascending, c12) and gate g:
        u_t      = x_t B_I                                   (per SwiGLU half m)
        z_{t,b}  = x_t W_I[:, b] + u_t C_I[:, b]             (the "XW + XBC" form)
        h~_{t,b} = g_{t,b} act(z_{t,b})
        q_t      = sum_b h~_{t,b} B_O[b, :]
        y_t      = sum_b h~_{t,b} W_O[b, :] + q_t C_O
    The backward holds W frozen (no dW_I / dW_O) and returns the LoRA factor
    gradients, dX, dgate and dW_R (the router is trained).

Storage convention (the library's, include/spt_ffn.h): w1 = W_I^T [m', D, d],
w2 = W_O [D, d]; b1 = B_I^T [m', r, d], c1 = C_I^T [m', D, r], b2 = B_O [D, r],
c2 = C_O [r, d].  m' = 2 for SwiGLU (gate, up), else 1 (arrays then carry a
leading axis of 1 here; the public functions accept either form).

Formulation: Algorithm 4 written as a loop over blocks with
token masks (numpy matmul as the GEMM step), with the LoRA terms kept
unmerged (x_t B_I first, then C_I) exactly as Eq. 5 writes them.  The pins
(tests/test_oracle_lora.py) compare it with the per-token C oracle
(spt_oracle.c) run on the MERGED weights W + BC, and the factor gradients with
the chain rule through that C oracle's full weight gradients
(dB = dW'... projections), plus central finite differences.
"""
from __future__ import annotations

import numpy as np

from . import ACT_GELU, ACT_RELU, ACT_SWIGLU, GATE_SIGMOID


def _sig(z):
    return 1.0 / (1.0 + np.exp(-z))


def _act(act, zg, zu):
    if act == ACT_RELU:
        return np.maximum(zg, 0.0)
    if act == ACT_GELU:
        from scipy.special import erf
        return 0.5 * zg * (1.0 + erf(zg / np.sqrt(2.0)))
    return zg * _sig(zg) * zu


def _act_grad(act, zg, zu, dh):
    """(dZg, dZu) for dh = dL/dact(z)."""
    if act == ACT_RELU:
        return dh * (zg > 0.0), None
    if act == ACT_GELU:
        from scipy.special import erf
        phi = np.exp(-0.5 * zg * zg) / np.sqrt(2.0 * np.pi)
        return dh * (0.5 * (1.0 + erf(zg / np.sqrt(2.0))) + zg * phi), None
    s = _sig(zg)
    return dh * zu * s * (1.0 + zg * (1.0 - s)), dh * zg * s


def _mp(act):
    return 2 if act == ACT_SWIGLU else 1


def _w1(w1, act):
    w1 = np.asarray(w1, np.float64)
    return w1.reshape((_mp(act),) + w1.shape[-2:])


def _lora(lora, act):
    mp = _mp(act)
    b1 = np.asarray(lora["b1"], np.float64)
    c1 = np.asarray(lora["c1"], np.float64)
    return (b1.reshape((mp,) + b1.shape[-2:]), c1.reshape((mp,) + c1.shape[-2:]),
            np.asarray(lora["b2"], np.float64), np.asarray(lora["c2"], np.float64))


def _blocks(logits, topk_idx, G, gate):
    """For block i (Alg. 4 line 1): the token mask (line 2) and the tokens' gates."""
    for i in range(G):
        mask = (topk_idx == i).any(axis=1)                       # eq(Indices, i)
        if mask.any():
            g = _sig(logits[mask, i]) if gate == GATE_SIGMOID else np.ones(int(mask.sum()))
            yield i, mask, g


def lora_forward(x, w1, w2, lora, logits, topk_idx, act, gate, want_stash=False):
    """y [T, d] of the LoRA-wrapped routed FFN (module docstring)."""
    x = np.asarray(x, np.float64)
    w1 = _w1(w1, act)
    w2 = np.asarray(w2, np.float64)
    b1, c1, b2, c2 = _lora(lora, act)
    lg = np.asarray(logits, np.float64)
    T, d = x.shape
    D, G = w2.shape[0], lg.shape[1]
    bw = D // G
    u = [x @ b1[m].T for m in range(w1.shape[0])]               # x B_I           [T, r]
    y = np.zeros((T, d))
    q = np.zeros((T, b2.shape[1]))
    for i, mask, g in _blocks(lg, topk_idx, G, gate):
        rows = slice(i * bw, (i + 1) * bw)
        X_i = x[mask]                                            # line 3
        z = [X_i @ w1[m, rows].T + u[m][mask] @ c1[m, rows].T    # X W_I + (X B_I) C_I
             for m in range(w1.shape[0])]
        H = g[:, None] * _act(act, z[0], z[-1])                  # line 4 (+ gate, c2)
        y[mask] += H @ w2[rows]                                  # line 5 (c1: accumulate)
        q[mask] += H @ b2[rows]                                  # h~ B_O
    y += q @ c2                                                  # (sum_b h~ B_O) C_O
    return (y, {"u": u, "q": q}) if want_stash else y


def lora_backward(x, w1, w2, w_r, lora, logits, topk_idx, dy, act, gate):
    """Gradients of <dy, y> with W_I, W_O frozen and routing fixed (c11):
    dict of dx [T,d], dgate [T,k] (ascending blocks), dw_r [G,d], db1, dc1, db2, dc2
    (shapes of the factors; db1/dc1 with the leading m' axis)."""
    x = np.asarray(x, np.float64)
    w1 = _w1(w1, act)
    w2 = np.asarray(w2, np.float64)
    w_r = np.asarray(w_r, np.float64)
    b1, c1, b2, c2 = _lora(lora, act)
    lg = np.asarray(logits, np.float64)
    dy = np.asarray(dy, np.float64)
    ti = np.asarray(topk_idx)
    T, d = x.shape
    D, G = w2.shape[0], lg.shape[1]
    k = ti.shape[1]
    bw = D // G
    mp = w1.shape[0]
    u = [x @ b1[m].T for m in range(mp)]
    v = dy @ c2.T                                                # dL/dq = dy C_O^T   [T, r]
    q = np.zeros((T, b2.shape[1]))
    du = [np.zeros_like(u[m]) for m in range(mp)]
    dx = np.zeros((T, d))
    dgate = np.zeros((T, k))
    dlogit = np.zeros((T, G))
    db1, dc1 = np.zeros_like(b1), np.zeros_like(c1)
    db2 = np.zeros_like(b2)
    for i, mask, g in _blocks(lg, ti, G, gate):
        rows = slice(i * bw, (i + 1) * bw)
        X_i = x[mask]
        z = [X_i @ w1[m, rows].T + u[m][mask] @ c1[m, rows].T for m in range(mp)]
        A = _act(act, z[0], z[-1])
        H = g[:, None] * A
        q[mask] += H @ b2[rows]
        # dL/dh~ = dy W_O[b]^T + (dy C_O^T) B_O[b]^T                 (h~ feeds both terms)
        dH = dy[mask] @ w2[rows].T + v[mask] @ b2[rows].T
        db2[rows] += H.T @ v[mask]                               # dL/dB_O[b] = h~^T (dy C_O^T)
        dg = (dH * A).sum(axis=1)                                # dL/dg
        dgate[mask, np.argmax(ti[mask] == i, axis=1)] = dg
        if gate == GATE_SIGMOID:
            dlogit[mask, i] = dg * g * (1.0 - g)
        dzg, dzu = _act_grad(act, z[0], z[-1], g[:, None] * dH)
        dz = [dzg] if mp == 1 else [dzg, dzu]
        for m in range(mp):
            dx[mask] += dz[m] @ w1[m, rows]                      # through X W_I
            du[m][mask] += dz[m] @ c1[m, rows]                   # through (X B_I) C_I
            dc1[m, rows] += dz[m].T @ u[m][mask]                 # dL/dC_I[:, b]^T
    for m in range(mp):
        dx += du[m] @ b1[m]                                      # u = x B_I
        db1[m] = du[m].T @ x                                     # dL/dB_I^T
    dc2 = q.T @ dy                                               # dL/dC_O = q^T dy
    dx += dlogit @ w_r                                           # router: x_R = x W_R
    dw_r = dlogit.T @ x
    return {"dx": dx, "dgate": dgate, "dw_r": dw_r, "db1": db1, "dc1": dc1, "db2": db2,
            "dc2": dc2}


def merged_weights(w1, w2, lora, act):
    """W_I + B_I C_I and W_O + B_O C_O in the library's storage (fp64): the
    "merge W' = W + BC" of PAPER.md:161, used by the pins only."""
    w1 = _w1(w1, act)
    b1, c1, b2, c2 = _lora(lora, act)
    w1m = np.stack([w1[m] + c1[m] @ b1[m] for m in range(w1.shape[0])])
    w2m = np.asarray(w2, np.float64) + b2 @ c2
    return (w1m if w1m.shape[0] == 2 else w1m[0]), w2m

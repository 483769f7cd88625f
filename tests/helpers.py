"""Shared test helpers: run the CUDA path (through the C ABI) and the oracle on
the same seeded inputs, and the error metric of SURVEY §8(c) reading c14."""
from __future__ import annotations

import json
import os

import numpy as np

import synthetic as S

TOL = {"f32": 1e-4, "bf16": 2e-2}   # BASELINE.json north_star: max relative error


def relerr(got, ref) -> float:
    """infinity-norm relative error  max|a - o| / max|o|  (reading c14)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.max(np.abs(ref)) if ref.size else 0.0
    if ref.size == 0:
        return 0.0
    err = float(np.max(np.abs(got - ref)) / max(den, 1e-30))
    _log_elementwise(got, ref, err)
    return err


def elemerr(got, ref, floor=1e-3) -> float:
    """Reading c14's companion metric: elementwise relative error with a floor,
    max_i |a_i - o_i| / max(|o_i|, floor * max|o|).  Errors confined to
    small-magnitude entries (one block's dw_r row, a low-gate pair) show up
    here although they hide under the infinity-norm bound's global max."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    den = np.maximum(np.abs(ref), floor * max(np.max(np.abs(ref)), 1e-30))
    return float(np.max(np.abs(got - ref) / den))


def relerr_rows(got, ref, floor=1e-3) -> float:
    """Per-row infinity-norm relative error (rows = the leading axis after
    flattening the rest), each row against its own max|o| floored at
    floor * (global max|o|); returns the worst row.  Used for per-block
    quantities (a block's dw rows, each block's dw_r row) so that one small
    block cannot hide under a large one."""
    got = np.asarray(got, np.float64).reshape(len(got), -1)
    ref = np.asarray(ref, np.float64).reshape(len(ref), -1)
    if ref.size == 0:
        return 0.0
    gmax = max(float(np.max(np.abs(ref))), 1e-30)
    den = np.maximum(np.max(np.abs(ref), axis=1), floor * gmax)
    return float(np.max(np.max(np.abs(got - ref), axis=1) / den))


_ERRLOG = os.environ.get("SPT_ERRLOG")  # optional JSON-lines log of both metrics per check


def _log_elementwise(got, ref, err):
    if not _ERRLOG:
        return
    test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    with open(_ERRLOG, "a") as f:
        f.write(json.dumps({"test": test, "shape": list(ref.shape), "inf_rel": err,
                            "elem_floored": elemerr(got, ref)}) + "\n")


def torch_dtype(cfg):
    import torch
    return torch.float32 if cfg.dtype == "f32" else torch.bfloat16


def to_dev(a, cfg):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch_dtype(cfg)).cuda()


def gpu_run(cfg: S.FfnConfig, T: int, inputs: dict, logits_in=None, backward=True,
            accumulate_from=None, want_dgate=True, balance_weight=0.0, deterministic=False):
    """Route -> forward -> backward through the ABI; returns numpy outputs
    (balance_weight: lambda of the load-balancing loss; adds "loss_lb";
    deterministic: SPT_FFN_DETERMINISTIC, the ascending-block k-way sums)."""
    import torch
    import paper_2312_10365_b200 as P
    f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, torch_dtype(cfg), cfg.act, cfg.gate,
                    balance_weight=balance_weight, deterministic=deterministic)
    x, w1, w2, w_r, dy = (to_dev(inputs[n], cfg) for n in ("x", "w1", "w2", "w_r", "dy"))
    flags = 0
    if logits_in is not None:
        f.route_buf.logits.copy_(torch.from_numpy(np.ascontiguousarray(logits_in, np.float32)))
        flags = P.SPT_ROUTE_LOGITS_IN
    f.route(x, w_r, flags)
    y = f.forward(x, w1, w2)
    out = {n: getattr(f.route_buf, n).cpu().numpy() for n in
           ("logits", "topk_idx", "topk_gate", "block_offsets", "bucket_token", "bucket_gate",
            "pair_slot", "tile_offsets")}
    out["y"] = y.float().cpu().numpy()
    out["loss_lb"] = float(f.balance_loss().cpu()[0])
    if backward:
        bflags = 0
        if accumulate_from is not None:
            f.dw1.copy_(torch.from_numpy(accumulate_from["dw1"]))
            f.dw2.copy_(torch.from_numpy(accumulate_from["dw2"]))
            f.dw_r.copy_(torch.from_numpy(accumulate_from["dw_r"]))
            bflags = P.SPT_BWD_ACCUMULATE_DW
        dx, dw1, dw2, dw_r = f.backward(x, w1, w2, w_r, dy, flags=bflags, want_dgate=want_dgate)
        out.update(dx=dx.float().cpu().numpy(), dw1=dw1.cpu().numpy(), dw2=dw2.cpu().numpy(),
                   dw_r=dw_r.cpu().numpy())
        if want_dgate:
            out["dgate"] = f.dgate.cpu().numpy()
    torch.cuda.synchronize()
    return out


def oracle_run(orc, cfg: S.FfnConfig, inputs: dict, logits, topk_idx, tokens=None, blocks=None,
               backward=True, lb_weight=0.0):
    """fp64 oracle on the same input bits.  logits: fp64 (or fp32) [T,G]."""
    y = orc.forward(inputs["x"], inputs["w1"], inputs["w2"], logits, topk_idx, cfg.act, cfg.gate,
                    tokens=tokens)
    out = {"y": y}
    if backward:
        out.update(orc.backward(inputs["x"], inputs["w1"], inputs["w2"], inputs["w_r"], logits,
                                topk_idx, inputs["dy"], cfg.act, cfg.gate, tokens=tokens, blocks=blocks,
                                lb_weight=lb_weight))
    return out


def relu_kink_fixup(cfg, inp, logits, topk_idx, got, ref, tokens=None, blocks=None, tau=1e-3):
    """ReLU's derivative is a decision taken in floating point: relu'(z) = [z > 0].
    Where |z| < tau (z from the inputs in fp64 here, independent of both sides)
    the GPU's fp32 z and the oracle's fp64 z may fall on different sides of the
    kink, and both derivatives are valid within rounding (DESIGN reading c24).
    For every such (token, block, unit) the flip changes dx[t] by
    g dA[t,u] w1[u] and dw1[u] by g dA[t,u] x[t]; per dx row / dw1 row this
    adds to ref the flips the GPU took (least squares of the residual on the
    row's flip terms, nearly orthogonal vectors: coefficient ~1 for a taken flip,
    ~0 otherwise), so the standard bound then checks everything else.  tau covers
    the split fp32 path's z error (~1e-4 absolute at d = 4096).
    Returns the number of ambiguous elements.  ReLU only; y and dgate are
    continuous at the kink and are not touched."""
    if cfg.act != S.ACT_RELU:
        return 0
    x = inp["x"].astype(np.float64)
    w1 = inp["w1"].astype(np.float64)
    w2 = inp["w2"].astype(np.float64)
    dy = inp["dy"].astype(np.float64)
    lg = np.asarray(logits, np.float64)
    T, k, bw = topk_idx.shape[0], topk_idx.shape[1], cfg.bw
    amb = []  # (t, unit, delta sign, g dA)
    tok_set = None if tokens is None else set(int(t) for t in tokens)
    blk_set = None if blocks is None else set(int(b) for b in blocks)
    for t in range(T):
        for j in range(k):
            b = int(topk_idx[t, j])
            if tok_set is not None and t not in tok_set and (blk_set is None or b not in blk_set):
                continue  # a pair no compared quantity depends on
            rows = slice(b * bw, (b + 1) * bw)
            z = w1[rows] @ x[t]
            near = np.nonzero(np.abs(z) < tau)[0]
            if not len(near):
                continue
            g = 1.0 / (1.0 + np.exp(-lg[t, b])) if cfg.gate == S.GATE_SIGMOID else 1.0
            da = w2[b * bw + near] @ dy[t]
            for u, a, zz in zip(near, da, z[near]):
                # the oracle used [z > 0]; the alternative removes / adds the term
                amb.append((t, b * bw + int(u), -1.0 if zz > 0 else 1.0, g * a))
    if not amb:
        return 0

    def best(gv, rv, terms):
        # least squares of the residual on the row's flip terms (a few nearly
        # orthogonal vectors): coefficient ~1 where the GPU took a flip, ~0 where not
        r = gv - rv
        V = np.stack([sgn * vec for sgn, vec in terms], axis=1)
        c = np.linalg.lstsq(V, r, rcond=None)[0]
        return rv + V @ (c > 0.5).astype(np.float64)

    if "dx" in ref:
        by_t = {}
        for t, u, sgn, gda in amb:
            if tok_set is None or t in tok_set:
                by_t.setdefault(t, []).append((sgn, gda * w1[u]))
        for t, terms in by_t.items():
            ref["dx"][t] = best(np.asarray(got["dx"][t], np.float64), ref["dx"][t], terms)
    if "dw1" in ref:
        by_u = {}
        for t, u, sgn, gda in amb:
            if blk_set is None or u // bw in blk_set:
                by_u.setdefault(u, []).append((sgn, gda * x[t]))
        for u, terms in by_u.items():
            ref["dw1"][u] = best(np.asarray(got["dw1"][u], np.float64), ref["dw1"][u], terms)
    return len(amb)

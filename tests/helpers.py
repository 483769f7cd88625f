"""Shared test helpers: run the CUDA path (through the C ABI) and the oracle on
the same seeded inputs, and the error metric of SURVEY §8(c) reading c14."""
from __future__ import annotations

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
    return float(np.max(np.abs(got - ref)) / max(den, 1e-30))


def torch_dtype(cfg):
    import torch
    return torch.float32 if cfg.dtype == "f32" else torch.bfloat16


def to_dev(a, cfg):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch_dtype(cfg)).cuda()


def gpu_run(cfg: S.FfnConfig, T: int, inputs: dict, logits_in=None, backward=True,
            accumulate_from=None, want_dgate=True, balance_weight=0.0):
    """Route -> forward -> backward through the ABI; returns numpy outputs
    (balance_weight: lambda of the load-balancing loss; adds "loss_lb")."""
    import torch
    import paper_2312_10365_b200 as P
    f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, torch_dtype(cfg), cfg.act, cfg.gate,
                    balance_weight=balance_weight)
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

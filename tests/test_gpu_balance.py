"""GPU parity of the load-balancing loss and its gradient (SURVEY §8(f) f2,
reading c18) against the fp64 oracle (pinned in test_oracle_balance.py).

Loss: spt_ffn_balance_loss on the GPU's own fp32 logits vs oracle.balance on
the same logits (fp32 softmax + fixed-order sums: relative 1e-5).  Gradient:
the full backward with lambda > 0 vs oracle.backward(lb_weight=lambda) -- the
balance term reaches dw_r and dx through every block's logit (with GATE_NONE
it is the router's only gradient); dw1, dw2, dgate are the task loss's.
Tolerances: 1e-4 fp32 / 2e-2 bf16 (reading c14).
"""
import numpy as np
import pytest

import synthetic as S
from helpers import TOL, gpu_run, oracle_run, relerr

pytestmark = pytest.mark.gpu

NAMES = ("y", "dx", "dw1", "dw2", "dw_r", "dgate")


def _run(orc, cfg, T, lam, kind=None):
    inp = S.make_inputs(cfg, T)
    logits = None if kind is None else S.make_logits(T, cfg.G, cfg.k, kind, seed=cfg.seed)
    got = gpu_run(cfg, T, inp, logits_in=logits, balance_weight=lam)
    # the oracle's own logits: the fixed ones, else its fp64 x W_R (never the GPU's)
    lg = logits.astype(np.float64) if logits is not None else orc.router(inp["x"], inp["w_r"])
    assert np.array_equal(got["topk_idx"], orc.topk(got["logits"], cfg.k))
    L, _ = orc.balance(lg, got["topk_idx"])
    assert abs(got["loss_lb"] - L) <= 1e-5 * max(1.0, abs(L)), (got["loss_lb"], L)
    ref = oracle_run(orc, cfg, inp, lg, got["topk_idx"], lb_weight=lam)
    tol = TOL[cfg.dtype]
    errs = {n: relerr(got[n], ref[n]) for n in NAMES}
    assert all(e <= tol for e in errs.values()), (cfg.name, errs)
    return got, ref


@pytest.mark.parametrize("gate", [S.GATE_SIGMOID, S.GATE_NONE])
@pytest.mark.parametrize("name,T", [("tiny", 300), ("bert", 700), ("llama", 300)])
def test_balance_gradient(orc, name, T, gate):
    _run(orc, S.CONFIGS[name].with_(gate=gate), T, lam=0.5)


@pytest.mark.parametrize("kind", ["zipf", "same"])
def test_balance_skewed_routing(orc, kind):
    """Skewed buckets (large f_g on a few blocks): the loss is far from 1."""
    got, _ = _run(orc, S.CONFIGS["opt"], 700, lam=0.3, kind=kind)
    assert got["loss_lb"] > 1.05


def test_balance_wide_blocks(orc):
    cfg = S.FfnConfig("wide_lb", 256, 2048, 4, 2, 500, "bf16", S.ACT_GELU)
    _run(orc, cfg, 500, lam=0.2)


def test_balance_loss_empty_batch():
    import torch
    import paper_2312_10365_b200 as P
    f = P.RoutedFFN(0, 128, 512, 8, 2, torch.bfloat16, P.SPT_ACT_RELU, balance_weight=0.1)
    x = torch.empty(0, 128, device="cuda", dtype=torch.bfloat16)
    f.route(x, torch.randn(8, 128, device="cuda", dtype=torch.bfloat16))
    f.loss_lb.fill_(7)
    assert float(f.balance_loss().cpu()[0]) == 0.0

"""CPU pin of the test helper relu_kink_fixup (tests/helpers.py, DESIGN reading
c24): given an oracle result and a 'device' result that took the other side of
the ReLU kink on a known subset of near-zero pre-activations, the fix-up must
recover exactly that subset -- and must not absorb any other deviation."""
import numpy as np

import oracle as orc
import synthetic as S
from helpers import oracle_run, relu_kink_fixup


def _case(tau):
    cfg = S.CONFIGS["tiny"]  # fp32, ReLU, sigmoid gate
    T = 96
    inp = S.make_inputs(cfg, T)
    lg = orc.router(inp["x"], inp["w_r"])
    ti = orc.topk(lg.astype(np.float32), cfg.k)
    ref = oracle_run(orc, cfg, inp, lg, ti)
    # the flip terms, computed independently here: for |z| < tau the other
    # derivative adds -+ g dA w1[u] to dx[t] and -+ g dA x[t] to dw1[u]
    x, w1, w2, dy = (inp[n].astype(np.float64) for n in ("x", "w1", "w2", "dy"))
    flips = []
    for t in range(T):
        for b in ti[t]:
            rows = np.arange(b * cfg.bw, (b + 1) * cfg.bw)
            z = w1[rows] @ x[t]
            g = 1 / (1 + np.exp(-lg[t, b]))
            for u in rows[np.abs(z) < tau]:
                s = -1.0 if w1[u] @ x[t] > 0 else 1.0
                flips.append((t, int(u), s * g * (w2[u] @ dy[t])))
    return cfg, inp, lg, ti, ref, x, w1, flips


def test_fixup_recovers_taken_flips():
    tau = 0.02
    cfg, inp, lg, ti, ref, x, w1, flips = _case(tau)
    assert len(flips) > 20
    rng = np.random.default_rng(0)
    taken = [f for f in flips if rng.random() < 0.5]
    dev = {"dx": ref["dx"].copy(), "dw1": ref["dw1"].copy()}
    for t, u, c in taken:
        dev["dx"][t] += c * w1[u]
        dev["dw1"][u] += c * x[t]
    fixed = {"dx": ref["dx"].copy(), "dw1": ref["dw1"].copy()}
    n = relu_kink_fixup(cfg, inp, lg, ti, dev, fixed, tau=tau)
    assert n == len(flips)
    assert np.max(np.abs(fixed["dx"] - dev["dx"])) < 1e-9
    assert np.max(np.abs(fixed["dw1"] - dev["dw1"])) < 1e-9


def test_fixup_does_not_absorb_other_errors():
    tau = 0.02
    cfg, inp, lg, ti, ref, x, w1, flips = _case(tau)
    dev = {"dx": ref["dx"].copy(), "dw1": ref["dw1"].copy()}
    t, u, c = flips[0]
    dev["dx"][t] += c * w1[u]          # a genuine kink flip
    dev["dx"][t + 1 if t + 1 < len(dev["dx"]) else 0, 3] += 0.5   # a bug elsewhere
    dev["dw1"][7, 5] -= 0.25                                       # and in dw1
    fixed = {"dx": ref["dx"].copy(), "dw1": ref["dw1"].copy()}
    relu_kink_fixup(cfg, inp, lg, ti, dev, fixed, tau=tau)
    assert np.max(np.abs(fixed["dx"] - dev["dx"])) >= 0.49
    assert np.max(np.abs(fixed["dw1"] - dev["dw1"])) >= 0.24

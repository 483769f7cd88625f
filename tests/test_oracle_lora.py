"""Pins for the oracle of the LoRA-wrapped routed FFN -- CPU only.

oracle/lora.py (numpy, Alg. 4 block loop, LoRA terms unmerged as Eq. 5 writes
them: XW + (XB)C) is checked against things other than itself:
  * the per-token C oracle (spt_oracle.c, already pinned) run on the MERGED
    weights W + BC -- the identity X(W + BC) = XW + XBC of PAPER.md:159 --
    for y, dx, dgate and dW_R;
  * the factor gradients against the chain rule through that C oracle's full
    weight gradients dW' at the merged weights: with W' = W + BC,
    dL/dB = dL/dW' C^T and dL/dC = B^T dL/dW' (in the library's transposed
    storage: db1 = c1^T dw1', dc1 = dw1' b1^T, db2 = dw2' c2^T, dc2 = b2^T dw2');
  * zero LoRA factors reduce it to the plain routed FFN;
  * k = G with gate NONE reduces it to the dense LoRA FFN
    act(X(W_I + B_I C_I))(W_O + B_O C_O), numpy matmul;
  * central finite differences in fp64 for every trained tensor (eps = 1e-6).
"""
import numpy as np
import pytest

import synthetic as S
from oracle import lora as OL
from test_oracle_ffn import dense_ffn, rel, small

ACTS = [S.ACT_RELU, S.ACT_GELU, S.ACT_SWIGLU]
GATES = [S.GATE_NONE, S.GATE_SIGMOID]


def factors(D, d, r, act, seed=5, scale=1.0):
    rng = np.random.default_rng(seed)
    lead = (2,) if act == S.ACT_SWIGLU else ()
    return {"b1": rng.standard_normal(lead + (r, d)) / np.sqrt(d),
            "c1": rng.standard_normal(lead + (D, r)) * 0.5 * scale,
            "b2": rng.standard_normal((D, r)) * 0.3,
            "c2": rng.standard_normal((r, d)) * 0.5 * scale}


def setup(act, gate, T=9, d=6, D=12, G=4, k=2, r=3, seed=3):
    import oracle as orc
    x, w1, w2, w_r, dy = small(T=T, d=d, D=D, G=G, k=k, act=act, seed=seed)
    lo = factors(D, d, r, act, seed=seed + 1)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), k)
    return x, w1, w2, w_r, dy, lo, lg, ti


@pytest.mark.parametrize("gate", GATES)
@pytest.mark.parametrize("act", ACTS)
def test_forward_equals_merged_weights(orc, act, gate):
    x, w1, w2, w_r, dy, lo, lg, ti = setup(act, gate)
    y = OL.lora_forward(x, w1, w2, lo, lg, ti, act, gate)
    w1m, w2m = OL.merged_weights(w1, w2, lo, act)
    ref = orc.forward(x, w1m, w2m, lg, ti, act, gate)
    assert rel(y, ref) < 1e-12
    # the LoRA terms are not negligible in this pin
    assert rel(orc.forward(x, w1, w2, lg, ti, act, gate), ref) > 1e-2


@pytest.mark.parametrize("gate", GATES)
@pytest.mark.parametrize("act", ACTS)
def test_backward_equals_chain_rule_through_merged_weights(orc, act, gate):
    x, w1, w2, w_r, dy, lo, lg, ti = setup(act, gate)
    g = OL.lora_backward(x, w1, w2, w_r, lo, lg, ti, dy, act, gate)
    w1m, w2m = OL.merged_weights(w1, w2, lo, act)
    ref = orc.backward(x, w1m, w2m, w_r, lg, ti, dy, act, gate)
    for n in ("dx", "dgate"):
        assert rel(g[n], ref[n]) < 1e-12, n
    if gate == S.GATE_SIGMOID:
        assert rel(g["dw_r"], ref["dw_r"]) < 1e-12
    else:
        assert np.all(g["dw_r"] == 0) and np.all(ref["dw_r"] == 0)
    mp = 2 if act == S.ACT_SWIGLU else 1
    dw1 = ref["dw1"].reshape((mp,) + ref["dw1"].shape[-2:])
    b1 = np.asarray(lo["b1"]).reshape((mp,) + lo["b1"].shape[-2:])
    c1 = np.asarray(lo["c1"]).reshape((mp,) + lo["c1"].shape[-2:])
    # w1' = w1 + c1 b1  =>  dL/db1 = c1^T dw1',  dL/dc1 = dw1' b1^T
    for m in range(mp):
        assert rel(g["db1"][m], c1[m].T @ dw1[m]) < 1e-12
        assert rel(g["dc1"][m], dw1[m] @ b1[m].T) < 1e-12
    # w2' = w2 + b2 c2  =>  dL/db2 = dw2' c2^T,  dL/dc2 = b2^T dw2'
    assert rel(g["db2"], ref["dw2"] @ lo["c2"].T) < 1e-12
    assert rel(g["dc2"], lo["b2"].T @ ref["dw2"]) < 1e-12


@pytest.mark.parametrize("act", ACTS)
def test_zero_factors_reduce_to_routed_ffn(orc, act):
    x, w1, w2, w_r, dy, lo, lg, ti = setup(act, S.GATE_SIGMOID)
    z = {n: np.zeros_like(v) for n, v in lo.items()}
    y = OL.lora_forward(x, w1, w2, z, lg, ti, act, S.GATE_SIGMOID)
    assert rel(y, orc.forward(x, w1, w2, lg, ti, act, S.GATE_SIGMOID)) < 1e-13
    # LoRA's usual init (C_I = 0, C_O = 0): still the routed FFN; B grads vanish, C grads do not
    lo0 = dict(lo, c1=np.zeros_like(lo["c1"]), c2=np.zeros_like(lo["c2"]))
    y0 = OL.lora_forward(x, w1, w2, lo0, lg, ti, act, S.GATE_SIGMOID)
    assert rel(y0, orc.forward(x, w1, w2, lg, ti, act, S.GATE_SIGMOID)) < 1e-13
    g = OL.lora_backward(x, w1, w2, w_r, lo0, lg, ti, dy, act, S.GATE_SIGMOID)
    assert np.all(g["db1"] == 0) and np.all(g["db2"] == 0)
    assert np.max(np.abs(g["dc1"])) > 1e-3 and np.max(np.abs(g["dc2"])) > 1e-3


@pytest.mark.parametrize("act", ACTS)
def test_k_equals_G_is_dense_lora_ffn(orc, act):
    T, d, D, G, r = 6, 5, 8, 4, 2
    x, w1, w2, w_r, dy = small(T=T, d=d, D=D, G=G, k=G, act=act, seed=8)
    lo = factors(D, d, r, act, seed=9)
    lg = orc.router(x, w_r)
    ti = np.tile(np.arange(G, dtype=np.int32), (T, 1))
    y = OL.lora_forward(x, w1, w2, lo, lg, ti, act, S.GATE_NONE)
    # PAPER.md:159  Y = X(W + BC) for both projections, written densely
    if act == S.ACT_SWIGLU:
        W_I = [w1[m].T + lo["b1"][m].T @ lo["c1"][m].T for m in range(2)]
        w1m = np.stack([W.T for W in W_I])
    else:
        w1m = (w1.T + lo["b1"].T @ lo["c1"].T).T
    W_O = w2 + lo["b2"] @ lo["c2"]
    assert rel(y, dense_ffn(x, w1m, W_O, act)) < 1e-12


def _loss(x, w1, w2, w_r, lo, ti, dy, act, gate):
    import oracle as orc
    lg = orc.router(x, w_r)
    return float(np.sum(dy * OL.lora_forward(x, w1, w2, lo, lg, ti, act, gate)))


@pytest.mark.parametrize("gate", GATES)
@pytest.mark.parametrize("act", ACTS)
def test_backward_matches_central_differences(orc, act, gate):
    T, d, D, G, k, r = 4, 5, 8, 4, 2, 2
    x, w1, w2, w_r, dy, lo, lg, ti = setup(act, gate, T=T, d=d, D=D, G=G, k=k, r=r, seed=21)
    if act == S.ACT_RELU:  # margin check: FD must not cross a kink
        w1m, _ = OL.merged_weights(w1, w2, lo, act)
        assert np.min(np.abs(x @ w1m.T)) > 1e-4
    an = OL.lora_backward(x, w1, w2, w_r, lo, lg, ti, dy, act, gate)
    eps = 1e-6
    params = {"x": x, "w_r": w_r, **lo}
    for name, gname in [("x", "dx"), ("w_r", "dw_r"), ("b1", "db1"), ("c1", "dc1"), ("b2", "db2"),
                        ("c2", "dc2")]:
        P = params[name]
        fd = np.zeros_like(P)
        it = np.nditer(P, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = P[idx]
            P[idx] = old + eps
            lp = _loss(params["x"], w1, w2, params["w_r"], lo, ti, dy, act, gate)
            P[idx] = old - eps
            lm = _loss(params["x"], w1, w2, params["w_r"], lo, ti, dy, act, gate)
            P[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        a = np.asarray(an[gname]).reshape(fd.shape)
        if gate == S.GATE_NONE and name == "w_r":
            assert np.all(a == 0) and np.max(np.abs(fd)) < 1e-8
            continue
        assert rel(a, fd) < 1e-6, (name, rel(a, fd))


def test_frozen_weights_have_no_gradient_output(orc):
    """LoRA freezes W: the backward returns no dW_I / dW_O."""
    x, w1, w2, w_r, dy, lo, lg, ti = setup(S.ACT_RELU, S.GATE_SIGMOID)
    g = OL.lora_backward(x, w1, w2, w_r, lo, lg, ti, dy, S.ACT_RELU, S.GATE_SIGMOID)
    assert set(g) == {"dx", "dgate", "dw_r", "db1", "dc1", "db2", "dc2"}


def test_synthetic_lora_shapes():
    cfg = S.CONFIGS["llama"]
    lo = S.make_lora(cfg, 16)
    assert lo["b1"].shape == (2, 16, cfg.d) and lo["c1"].shape == (2, cfg.D, 16)
    assert lo["b2"].shape == (cfg.D, 16) and lo["c2"].shape == (16, cfg.d)
    cfg = S.CONFIGS["bert"]
    lo = S.make_lora(cfg, 8)
    assert lo["b1"].shape == (8, cfg.d) and lo["c1"].shape == (cfg.D, 8)
    S.bf16_bits(lo["c1"])  # exactly representable in the storage dtype


@pytest.mark.parametrize("act", ACTS)
def test_rescaling_invariance(orc, act):
    """y is unchanged under B -> sB, C -> C/s, so <dB, B> = <dC, C> for both
    projections (used as a full-size GPU check of dB_I and dC_O)."""
    x, w1, w2, w_r, dy, lo, lg, ti = setup(act, S.GATE_SIGMOID)
    g = OL.lora_backward(x, w1, w2, w_r, lo, lg, ti, dy, act, S.GATE_SIGMOID)
    for a, b in (("b1", "c1"), ("b2", "c2")):
        lhs = float(np.sum(g["d" + a] * np.asarray(lo[a]).reshape(g["d" + a].shape)))
        rhs = float(np.sum(g["d" + b] * np.asarray(lo[b]).reshape(g["d" + b].shape)))
        assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(lhs)), (a, lhs, rhs)
        assert abs(lhs) > 1e-3

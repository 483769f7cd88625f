"""Pins for the oracle's routed-FFN forward and backward -- CPU only.

The oracle (O2, per-token, plain C) is checked against things other than
itself:
  * a hand-derived worked example (tests/golden/hand_ffn_example.json);
  * the textbook special case k = G, gate NONE == dense FFN Eq. 4 (PAPER.md:144,
    SPEC S:336) computed with numpy matmul;
  * k = G, gate SIGMOID == dense FFN with sigma-scaled hidden blocks;
  * O1 masked-dense (numpy, Fig. 6a) and O3 Alg.4-literal
     formulations;
  * a single token activating block 0 only == dense FFN with W zeroed outside
    block 0;
  * central finite differences in fp64 (eps=1e-6, rel err < 1e-6);
  * Euler homogeneity identities (no second implementation involved);
  * token-permutation equivariance; exact FLOP ratio beta.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import erf

import synthetic as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ACTS = [S.ACT_RELU, S.ACT_GELU, S.ACT_SWIGLU]
GATES = [S.GATE_NONE, S.GATE_SIGMOID]


def small(T=7, d=6, D=12, G=4, k=2, act=S.ACT_RELU, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, d))
    w1 = rng.standard_normal((2, D, d) if act == S.ACT_SWIGLU else (D, d)) / np.sqrt(d)
    w2 = rng.standard_normal((D, d)) / np.sqrt(k * D / G)
    w_r = rng.standard_normal((G, d)) / np.sqrt(d)
    dy = rng.standard_normal((T, d))
    return x, w1, w2, w_r, dy


def dense_act(act, zg, zu=None):
    if act == S.ACT_RELU:
        return np.maximum(zg, 0)
    if act == S.ACT_GELU:
        return 0.5 * zg * (1 + erf(zg / math.sqrt(2)))
    return zg / (1 + np.exp(-zg)) * zu


def dense_ffn(x, w1, w2, act, scale=None):
    """Eq. 4: Y = act(X W_I) W_O with W_I = w1^T, W_O = w2 (numpy matmul)."""
    if act == S.ACT_SWIGLU:
        H = dense_act(act, x @ w1[0].T, x @ w1[1].T)
    else:
        H = dense_act(act, x @ w1.T)
    if scale is not None:
        H = H * scale
    return H @ w2


def masked_dense(x, w1, w2, logits, ti, act, gate):
    """O1: M (.) act(X W_I) W_O with M[t,i] = g_{t,b(i)} if b(i) in S_t else 0."""
    T = x.shape[0]
    G = logits.shape[1]
    D = w2.shape[0]
    bw = D // G
    M = np.zeros((T, D))
    for t in range(T):
        for b in ti[t]:
            g = 1 / (1 + np.exp(-logits[t, b])) if gate == S.GATE_SIGMOID else 1.0
            M[t, b * bw:(b + 1) * bw] = g
    return dense_ffn(x, w1, w2, act, scale=M)


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("gate", GATES)
def test_hand_example(orc, gate):
    g = json.load(open(os.path.join(GOLD, "hand_ffn_example.json")))
    x, w1, w2, w_r, dy = (np.array(g[n], float) for n in ("x", "w1", "w2", "w_r", "dy"))
    lg = orc.router(x, w_r)
    assert lg.tolist() == [[1.0, -2.0]]
    ti = orc.topk(lg.astype(np.float32), 1)
    assert ti.tolist() == g["selected"]
    y = orc.forward(x, w1, w2, lg, ti, S.ACT_RELU, gate)
    bw_ = orc.backward(x, w1, w2, w_r, lg, ti, dy, S.ACT_RELU, gate)
    if gate == S.GATE_NONE:
        e = g["none"]
        for name, got in [("y", y), ("dx", bw_["dx"]), ("dgate", bw_["dgate"]), ("dw1", bw_["dw1"]),
                          ("dw2", bw_["dw2"]), ("dw_r", bw_["dw_r"])]:
            assert np.allclose(got, np.array(e[name], float), rtol=0, atol=1e-12), name
    else:
        e = g["sigmoid_in_terms_of_g"]
        gg = 1.0 / (1.0 + math.exp(2.0))
        dl = e["dlogit_over_g1mg"] * gg * (1 - gg)
        assert np.allclose(y, gg * np.array(e["y_over_g"]), atol=1e-14)
        assert np.allclose(bw_["dgate"], e["dgate"], atol=1e-12)
        assert np.allclose(bw_["dw1"], gg * np.array(e["dw1_over_g"]), atol=1e-14)
        assert np.allclose(bw_["dw2"], gg * np.array(e["dw2_over_g"]), atol=1e-14)
        assert np.allclose(bw_["dw_r"], dl * np.array(e["dw_r_over_dlogit"]), atol=1e-14)
        dx = gg * np.array(e["dx_ffn_over_g"]) + dl * np.array(e["dx_router_over_dlogit"])
        assert np.allclose(bw_["dx"], dx, atol=1e-14)


# ------------------------------------------------- special cases / forms
@pytest.mark.parametrize("act", ACTS)
def test_k_equals_G_gate_none_is_dense_ffn(orc, act):
    x, w1, w2, w_r, _ = small(act=act, G=4, k=4)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), 4)
    assert np.array_equal(ti, np.tile(np.arange(4), (x.shape[0], 1)))
    y = orc.forward(x, w1, w2, lg, ti, act, S.GATE_NONE)
    assert rel(y, dense_ffn(x, w1, w2, act)) < 1e-13


@pytest.mark.parametrize("act", ACTS)
def test_k_equals_G_sigmoid_is_scaled_dense(orc, act):
    G = 4
    x, w1, w2, w_r, _ = small(act=act, G=G, k=G)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), G)
    bw = w2.shape[0] // G
    scale = np.repeat(1 / (1 + np.exp(-lg)), bw, axis=1)
    y = orc.forward(x, w1, w2, lg, ti, act, S.GATE_SIGMOID)
    assert rel(y, dense_ffn(x, w1, w2, act, scale=scale)) < 1e-13


@pytest.mark.parametrize("act", ACTS)
@pytest.mark.parametrize("gate", GATES)
@pytest.mark.parametrize("G,k", [(4, 1), (4, 2), (6, 3)])
def test_three_formulations_agree(orc, act, gate, G, k):
    x, w1, w2, w_r, _ = small(T=11, d=5, D=G * 3, G=G, k=k, act=act)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), k)
    y2 = orc.forward(x, w1, w2, lg, ti, act, gate)
    y1 = masked_dense(x, w1, w2, lg, ti, act, gate)
    y3 = orc.alg4_forward(x, w1, w2, lg, ti, act, gate)
    assert rel(y2, y1) < 1e-12
    assert rel(y2, y3) < 1e-12


def test_single_token_block0_only(orc):
    """one token activating block 0 only, gate 1 == dense FFN with
    W_I, W_O zeroed outside block 0."""
    x, w1, w2, _, _ = small(T=1, d=6, D=12, G=4, k=1)
    lg = np.array([[9.0, 0.1, -0.2, 0.3]])
    ti = orc.topk(lg.astype(np.float32), 1)
    assert ti.tolist() == [[0]]
    y = orc.forward(x, w1, w2, lg, ti, S.ACT_RELU, S.GATE_NONE)
    w1z, w2z = np.zeros_like(w1), np.zeros_like(w2)
    w1z[:3], w2z[:3] = w1[:3], w2[:3]
    assert rel(y, dense_ffn(x, w1z, w2z, S.ACT_RELU)) < 1e-14


def test_token_subset_rows_equal_full(orc):
    x, w1, w2, w_r, dy = small(T=9, act=S.ACT_SWIGLU)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), 2)
    full = orc.forward(x, w1, w2, lg, ti, S.ACT_SWIGLU, S.GATE_SIGMOID)
    sub = orc.forward(x, w1, w2, lg, ti, S.ACT_SWIGLU, S.GATE_SIGMOID, tokens=[4, 1])
    assert np.array_equal(sub[[1, 4]], full[[1, 4]])
    assert np.isnan(sub[0]).all()
    bf = orc.backward(x, w1, w2, w_r, lg, ti, dy, S.ACT_SWIGLU, S.GATE_SIGMOID)
    bs = orc.backward(x, w1, w2, w_r, lg, ti, dy, S.ACT_SWIGLU, S.GATE_SIGMOID, tokens=[3], blocks=[2])
    assert np.array_equal(bs["dx"][3], bf["dx"][3])
    assert np.array_equal(bs["dw2"][6:9], bf["dw2"][6:9])
    assert np.array_equal(bs["dw1"][:, 6:9], bf["dw1"][:, 6:9])
    assert np.array_equal(bs["dw_r"][2], bf["dw_r"][2])


# ------------------------------------------------------ finite differences
def _loss(orc, x, w1, w2, w_r, dy, ti, act, gate):
    lg = x @ w_r.T       # logits recomputed from (x, w_r) so dx/dw_r see the gate path
    return float(np.sum(dy * orc.forward(x, w1, w2, lg, ti, act, gate)))


@pytest.mark.parametrize("act", ACTS)
@pytest.mark.parametrize("gate", GATES)
def test_backward_matches_central_differences(orc, act, gate):
    T, d, D, G, k = 4, 5, 8, 4, 2
    x, w1, w2, w_r, dy = small(T=T, d=d, D=D, G=G, k=k, act=act, seed=11)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), k)      # routing held fixed (reading c11)
    if act == S.ACT_RELU:                         # margin check: FD must not cross a kink
        z = x @ w1.T
        assert np.min(np.abs(z)) > 1e-4
    an = orc.backward(x, w1, w2, w_r, lg, ti, dy, act, gate)
    eps = 1e-6
    params = {"x": x, "w1": w1, "w2": w2, "w_r": w_r}
    for name, grad_name in [("x", "dx"), ("w1", "dw1"), ("w2", "dw2"), ("w_r", "dw_r")]:
        P = params[name]
        fd = np.zeros_like(P)
        it = np.nditer(P, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = P[idx]
            P[idx] = old + eps
            lp = _loss(orc, params["x"], params["w1"], params["w2"], params["w_r"], dy, ti, act, gate)
            P[idx] = old - eps
            lm = _loss(orc, params["x"], params["w1"], params["w2"], params["w_r"], dy, ti, act, gate)
            P[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        if gate == S.GATE_NONE and name == "w_r":
            assert np.all(an[grad_name] == 0) and np.max(np.abs(fd)) < 1e-8
            continue
        assert rel(an[grad_name], fd) < 1e-6, (name, rel(an[grad_name], fd))
    # dgate = dL/dg per pair: with SIGMOID, dL/dlogit_{t,b} = dgate g (1-g)
    if gate == S.GATE_SIGMOID:
        for t in range(T):
            for j, b in enumerate(ti[t]):
                lgp, lgm = lg.copy(), lg.copy()
                lgp[t, b] += eps
                lgm[t, b] -= eps
                fp = np.sum(dy * orc.forward(x, w1, w2, lgp, ti, act, gate))
                fm = np.sum(dy * orc.forward(x, w1, w2, lgm, ti, act, gate))
                g = 1 / (1 + np.exp(-lg[t, b]))
                assert abs((fp - fm) / (2 * eps) - an["dgate"][t, j] * g * (1 - g)) < 1e-7


# ---------------------------------------------------------------- identities
@pytest.mark.parametrize("act", ACTS)
@pytest.mark.parametrize("gate", GATES)
def test_euler_identities(orc, act, gate):
    x, w1, w2, w_r, dy = small(T=13, d=7, D=18, G=6, k=3, act=act, seed=5)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), 3)
    y = orc.forward(x, w1, w2, lg, ti, act, gate)
    g_ = orc.backward(x, w1, w2, w_r, lg, ti, dy, act, gate)
    dyy = float(np.sum(dy * y))
    # Y linear in W_O -> <dW2, W2> = <dY, Y>
    assert abs(np.sum(g_["dw2"] * w2) - dyy) < 1e-12 * max(1, abs(dyy))
    # Y linear in each gate -> sum_{t,j} g dgate = <dY, Y>
    gm = (1 / (1 + np.exp(-np.take_along_axis(lg, ti, 1)))) if gate == S.GATE_SIGMOID else 1.0
    assert abs(np.sum(gm * g_["dgate"]) - dyy) < 1e-12 * max(1, abs(dyy))
    if act == S.ACT_RELU:
        # ReLU FFN is degree-1 homogeneous in W_I
        assert abs(np.sum(g_["dw1"] * w1) - dyy) < 1e-12 * max(1, abs(dyy))
        if gate == S.GATE_NONE:   # ... and in X (gate path absent)
            assert abs(np.sum(g_["dx"] * x) - dyy) < 1e-12 * max(1, abs(dyy))
    if act == S.ACT_SWIGLU:
        # linear in the up projection
        assert abs(np.sum(g_["dw1"][1] * w1[1]) - dyy) < 1e-12 * max(1, abs(dyy))


def test_token_permutation_equivariance(orc):
    act, gate = S.ACT_GELU, S.GATE_SIGMOID
    x, w1, w2, w_r, dy = small(T=10, act=act, seed=8)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), 2)
    p = np.random.default_rng(0).permutation(10)
    a = orc.backward(x, w1, w2, w_r, lg, ti, dy, act, gate)
    b = orc.backward(x[p], w1, w2, w_r, lg[p], ti[p], dy[p], act, gate)
    ya = orc.forward(x, w1, w2, lg, ti, act, gate)
    yb = orc.forward(x[p], w1, w2, lg[p], ti[p], act, gate)
    assert rel(yb, ya[p]) < 1e-14 and rel(b["dx"], a["dx"][p]) < 1e-14
    for n in ("dw1", "dw2", "dw_r"):
        assert rel(b[n], a[n]) < 1e-13


@pytest.mark.parametrize("act", ACTS)
def test_flop_ratio_is_beta(orc, act):
    """n tokens, G=4, G'=2 -> flops = 0.5 x dense exactly."""
    T, d, D, G, k = 64, 32, 128, 4, 2
    mp = 2 if act == S.ACT_SWIGLU else 1
    dense = 2.0 * T * (mp + 1) * d * D
    assert orc.forward_gemm_flops(T, d, D, G, k, act) / dense == 0.5
    assert orc.forward_gemm_flops(T, 4096, 11008, 86, 22, act) / (2.0 * T * (mp + 1) * 4096 * 11008) \
        == pytest.approx(22 / 86, rel=1e-15)

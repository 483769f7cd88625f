"""Pins for the oracle's load-balancing loss -- CPU only.

L = G sum_g f_g pbar_g (reading c18: f_g = n_g / (T k)),
pinned against things other than its own formula:
  * SPEC's worked values: perfectly uniform routing and probabilities give
    exactly 1 ("G*G*(1/G)*(1/G)"); all tokens on one block with
    probability -> 1 approaches G;
  * the softmax Jacobian's invariant: each row of dL/dx_R sums to 0;
  * central finite differences in fp64 of L (routing held fixed, reading c11);
  * the full backward with lambda > 0: dW_R and dX of <dY, Y> + lambda L against
    central differences through x_R = x W_R.
"""
import numpy as np
import pytest

import synthetic as S
from test_oracle_ffn import rel, small


@pytest.mark.parametrize("G,k", [(8, 1), (8, 2), (4, 4), (86, 22)])
def test_uniform_routing_gives_exactly_one(orc, G, k):
    T = G  # token t activates blocks t, t+1, ..., t+k-1 (mod G): every block k times
    ti = np.sort(np.array([[(t + j) % G for j in range(k)] for t in range(T)]), axis=1)
    L, dl = orc.balance(np.full((T, G), 0.37), ti)
    assert abs(L - 1.0) < 1e-12
    assert np.max(np.abs(dl)) < 1e-15  # f_j - sum_g f_g p_g = 0 at the uniform point


@pytest.mark.parametrize("G", [2, 8, 86])
def test_one_block_limit_approaches_G(orc, G):
    T = 5
    lg = np.zeros((T, G))
    lg[:, 0] = 60.0  # p_t0 = 1 - (G-1) e^-60
    L, _ = orc.balance(lg, np.zeros((T, 1), dtype=np.int32))
    assert abs(L - G) < 1e-20 * G + G * (G - 1) * np.exp(-60.0) * 2


def test_gradient_rows_sum_to_zero(orc):
    rng = np.random.default_rng(1)
    T, G, k = 9, 7, 3
    lg = rng.standard_normal((T, G)) * 2
    ti = np.sort(np.argsort(-np.abs(lg), axis=1)[:, :k], axis=1).astype(np.int32)
    _, dl = orc.balance(lg, ti)
    assert np.max(np.abs(dl.sum(axis=1))) < 1e-15


def test_k_equals_G_is_constant_one(orc):
    """k = G: every f_g = 1/G, so L = sum_g pbar_g = 1 for any logits, gradient 0."""
    rng = np.random.default_rng(5)
    T, G = 4, 5
    L, dl = orc.balance(rng.standard_normal((T, G)) * 3, np.tile(np.arange(G), (T, 1)))
    assert abs(L - 1.0) < 1e-14 and np.max(np.abs(dl)) < 1e-15


@pytest.mark.parametrize("T,G,k", [(6, 4, 2), (11, 8, 3), (3, 5, 4)])
def test_gradient_matches_central_differences(orc, T, G, k):
    rng = np.random.default_rng(T * 100 + G)
    lg = rng.standard_normal((T, G)) * 1.5
    ti = np.sort(np.argsort(-np.abs(lg), axis=1)[:, :k], axis=1).astype(np.int32)
    _, dl = orc.balance(lg, ti)
    eps = 1e-6
    fd = np.zeros_like(lg)
    for t in range(T):
        for j in range(G):
            p, m = lg.copy(), lg.copy()
            p[t, j] += eps
            m[t, j] -= eps
            fd[t, j] = (orc.balance(p, ti, want_grad=False)[0] - orc.balance(m, ti, want_grad=False)[0]) / (2 * eps)
    assert rel(dl, fd) < 1e-6


@pytest.mark.parametrize("gate", [S.GATE_SIGMOID, S.GATE_NONE])
def test_backward_with_balance_matches_central_differences(orc, gate):
    T, d, D, G, k, lam = 5, 4, 8, 4, 2, 0.37
    act = S.ACT_GELU
    x, w1, w2, w_r, dy = small(T=T, d=d, D=D, G=G, k=k, act=act, seed=21)
    lg = orc.router(x, w_r)
    ti = orc.topk(lg.astype(np.float32), k)  # routing held fixed (reading c11)

    def loss(x_, w_r_):
        lg_ = x_ @ w_r_.T
        task = float(np.sum(dy * orc.forward(x_, w1, w2, lg_, ti, act, gate)))
        return task + lam * orc.balance(lg_, ti, want_grad=False)[0]

    an = orc.backward(x, w1, w2, w_r, lg, ti, dy, act, gate, lb_weight=lam)
    base = orc.backward(x, w1, w2, w_r, lg, ti, dy, act, gate)
    eps = 1e-6
    for name, P, grad in (("x", x, "dx"), ("w_r", w_r, "dw_r")):
        fd = np.zeros_like(P)
        it = np.nditer(P, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            old = P[idx]
            P[idx] = old + eps
            lp = loss(x, w_r)
            P[idx] = old - eps
            lm = loss(x, w_r)
            P[idx] = old
            fd[idx] = (lp - lm) / (2 * eps)
        assert rel(an[grad], fd) < 1e-6, (name, rel(an[grad], fd))
    # the balance term reaches the router even with GATE_NONE, and only dX / dW_R change
    assert np.max(np.abs(an["dw_r"] - base["dw_r"])) > 1e-3
    for n in ("dw1", "dw2", "dgate"):
        assert np.array_equal(an[n], base[n])

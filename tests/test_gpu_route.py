"""GPU parity of routing (a1 router, a2 top-k, a3 bucketing) against the oracle.

Top-k and bucket layouts must match BIT-EXACTLY on the same fp32 logits
(SPT_ROUTE_LOGITS_IN with generator-made logits, reading c15).  Router logits
computed on the GPU are compared with the oracle's fp64 x W_R within the
dtype's relative tolerance, and the GPU's selection is checked against the
oracle's wherever the k-th/(k+1)-th |logit| margin exceeds the logit error.
"""
import numpy as np
import pytest

import synthetic as S
from helpers import TOL, gpu_run, relerr

pytestmark = pytest.mark.gpu

ROUTE_CASES = [  # (T, G, k)
    (1, 8, 2), (255, 8, 2), (256, 8, 2), (257, 8, 1), (1000, 32, 8), (4099, 64, 16),
    (2050, 86, 22), (300, 4, 4), (513, 256, 8), (77, 256, 256), (1024, 5, 3),
]
KINDS = ["normal", "zipf", "same", "ties", "signed0"]


def _cfg(G, k, T, dtype="f32"):
    return S.FfnConfig("route", 64, G * 16, G, k, T, dtype, S.ACT_RELU)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("T,G,k", ROUTE_CASES)
def test_topk_and_buckets_bit_exact(orc, kind, T, G, k):
    cfg = _cfg(G, k, T)
    logits = S.make_logits(T, G, k, kind, seed=cfg.seed + T)
    inp = S.make_inputs(cfg, T)
    got = gpu_run(cfg, T, inp, logits_in=logits, backward=False)
    ti = orc.topk(logits, k)
    ref = orc.bucket(ti, G, tile_m=128)
    assert np.array_equal(got["topk_idx"], ti)
    for n in ("block_offsets", "bucket_token", "pair_slot", "tile_offsets"):
        assert np.array_equal(got[n], ref[n]), n
    # gates: sigmoid of the selected logit (fp32 on the GPU)
    sel = np.take_along_axis(logits.astype(np.float64), ti, 1)
    g_ref = 1.0 / (1.0 + np.exp(-sel))
    assert np.max(np.abs(got["topk_gate"] - g_ref)) < 1e-6
    assert np.array_equal(got["bucket_gate"][got["pair_slot"]], got["topk_gate"].reshape(-1))


def test_gate_none_gates_are_one(orc):
    cfg = _cfg(8, 2, 300).with_(gate=S.GATE_NONE)
    logits = S.make_logits(300, 8, 2, "normal")
    got = gpu_run(cfg, 300, S.make_inputs(cfg, 300), logits_in=logits, backward=False)
    assert np.all(got["topk_gate"] == 1.0) and np.all(got["bucket_gate"] == 1.0)


@pytest.mark.parametrize("name", ["tiny", "bert", "opt", "llama"])
def test_router_logits_and_selection(orc, name):
    cfg = S.CONFIGS[name]
    T = 1000
    inp = S.make_inputs(cfg, T)
    got = gpu_run(cfg, T, inp, backward=False)
    ref = orc.router(inp["x"], inp["w_r"])
    err = relerr(got["logits"], ref)
    assert err < (1e-5 if cfg.dtype == "f32" else 1e-4), err
    # selection: bit-exact on the GPU's own logits ...
    assert np.array_equal(got["topk_idx"], orc.topk(got["logits"], cfg.k))
    # ... and equal to the oracle's fp64-logit selection wherever the margin is safe
    ref_sel = orc.topk(ref.astype(np.float32), cfg.k)
    srt = np.sort(np.abs(ref), axis=1)[:, ::-1]
    margin = srt[:, cfg.k - 1] - (srt[:, cfg.k] if cfg.k < cfg.G else 0)
    bound = 4 * np.max(np.abs(got["logits"] - ref))
    safe = margin > bound
    assert safe.mean() > 0.95
    assert np.array_equal(got["topk_idx"][safe], ref_sel[safe])

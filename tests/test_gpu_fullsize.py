"""GPU parity at BASELINE.json's full sizes (in the launch configuration bench.py
times), on outputs the oracle can compute one by one:
  * routing: top-k bit-exact against the oracle on the GPU's own fp32 logits,
    bucket layout bit-exact against the oracle's bucketing of that top-k;
  * sampled token rows of y, dx and dgate (oracle per-token O2 form);
  * sampled blocks' rows of dw1, dw2, dw_r (oracle per-block backward, which
    sums over every token of T that activated the block);
  * properties that hold at any size, on the full GPU outputs: Euler identities
    <dW2, W2> = <dY, Y> and sum g*dgate = <dY, Y> (Y linear in W_O and in the gates).
Tolerance: bf16 2e-2 / fp32 1e-4 infinity-norm relative (reading c14).
"""
import numpy as np
import pytest

import synthetic as S
from helpers import TOL, gpu_run, relerr

pytestmark = pytest.mark.gpu

# (config, sampled blocks): LLaMA-size blocks are sampled once (each takes the
# oracle ~10 s single-threaded: it sums over all ~8k tokens of the block)
CASES = [("tiny", 2), ("bert", 2), ("opt", 2), ("llama", 1), ("llama_scale", 1),
         # the paper's own G = 8, beta = 1/2 workloads (wide blocks)
         ("opt2048_g8", 1), ("llama4096_g8", 1)]


@pytest.mark.parametrize("name,n_blocks", CASES)
def test_fullsize_sampled_parity(orc, name, n_blocks):
    cfg = S.ALL_CONFIGS[name]
    T = cfg.T
    inp = S.make_inputs(cfg, T)
    got = gpu_run(cfg, T, inp)

    # routing, bit-exact on the GPU's fp32 logits
    ti = orc.topk(got["logits"], cfg.k)
    assert np.array_equal(got["topk_idx"], ti)
    bref = orc.bucket(ti, cfg.G, tile_m=128)
    for n in ("block_offsets", "bucket_token", "pair_slot", "tile_offsets"):
        assert np.array_equal(got[n], bref[n]), n

    rng = np.random.default_rng(cfg.seed)
    tokens = np.unique(np.concatenate([[0, T - 1], rng.integers(0, T, 14)])).astype(np.int64)
    blocks = np.unique(rng.integers(0, cfg.G, n_blocks)).astype(np.int32)
    lg = got["logits"].astype(np.float64)   # same selection; gates from the same logits
    tol = TOL[cfg.dtype]

    y = orc.forward(inp["x"], inp["w1"], inp["w2"], lg, ti, cfg.act, cfg.gate, tokens=tokens)
    assert relerr(got["y"][tokens], y[tokens]) <= tol
    bw_ = orc.backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, inp["dy"], cfg.act,
                       cfg.gate, tokens=tokens, blocks=blocks)
    assert relerr(got["dx"][tokens], bw_["dx"][tokens]) <= tol
    assert relerr(got["dgate"][tokens], bw_["dgate"][tokens]) <= tol
    bwid = cfg.bw
    rows = np.concatenate([np.arange(b * bwid, (b + 1) * bwid) for b in blocks])
    if cfg.mprime == 2:
        assert relerr(got["dw1"][:, rows], bw_["dw1"][:, rows]) <= tol
    else:
        assert relerr(got["dw1"][rows], bw_["dw1"][rows]) <= tol
    assert relerr(got["dw2"][rows], bw_["dw2"][rows]) <= tol
    assert relerr(got["dw_r"][blocks], bw_["dw_r"][blocks]) <= tol

    # Euler identities on the full-size GPU outputs (fp64 reductions)
    dyy = float(np.sum(inp["dy"].astype(np.float64) * got["y"].astype(np.float64)))
    w2dw2 = float(np.sum(inp["w2"].astype(np.float64) * got["dw2"].astype(np.float64)))
    g = got["topk_gate"].astype(np.float64)
    gdg = float(np.sum(g * got["dgate"].astype(np.float64)))
    scale = float(np.sqrt(np.sum(inp["dy"].astype(np.float64) ** 2) * np.sum(got["y"].astype(np.float64) ** 2)))
    assert abs(w2dw2 - dyy) <= tol * scale
    assert abs(gdg - dyy) <= tol * scale

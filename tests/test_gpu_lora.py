"""GPU parity of the LoRA-wrapped routed FFN (ABI 3) against
the fp64 oracle (oracle/lora.py, pinned in test_oracle_lora.py).

Same protocol as test_gpu_ffn.py: seeded synthetic inputs plus seeded LoRA
factors (synthetic.make_lora), the GPU's own routing (its top-k checked equal to
the oracle's on the same fp32 logits), infinity-norm relative error <= 2e-2
(bf16, reading c14) on y, dx, dgate, dw_r and the four factor gradients.  Sizes
span several 128-row tiles with ragged tails; the BASELINE shapes (d, D, G, k)
at a few hundred tokens.
"""
import numpy as np
import pytest

import synthetic as S
from helpers import TOL, relerr, to_dev
from oracle import lora as OL

pytestmark = pytest.mark.gpu

NAMES = ("y", "dx", "dgate", "dw_r", "db1", "dc1", "db2", "dc2")


def gpu_run_lora(cfg, T, inp, lora, rank, balance_weight=0.0, accumulate_from=None):
    import torch
    import paper_2312_10365_b200 as P
    f = P.RoutedLoRAFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, torch.bfloat16, cfg.act, rank, cfg.gate,
                        balance_weight=balance_weight)
    x, w1, w2, w_r, dy = (to_dev(inp[n], cfg) for n in ("x", "w1", "w2", "w_r", "dy"))
    lo = {n: to_dev(v, cfg) for n, v in lora.items()}
    f.route(x, w_r)
    y = f.forward(x, w1, w2, lo)
    out = {"logits": f.route_buf.logits.cpu().numpy(), "topk_idx": f.route_buf.topk_idx.cpu().numpy(),
           "y": y.float().cpu().numpy()}
    flags = 0
    if accumulate_from is not None:
        for n, v in accumulate_from.items():
            (f.dw_r if n == "dw_r" else f.grads[n]).copy_(torch.from_numpy(np.ascontiguousarray(v, np.float32)))
        flags = P.SPT_BWD_ACCUMULATE_DW
    dx, grads, dw_r = f.backward(x, w1, w2, w_r, lo, dy, flags=flags, want_dgate=True)
    out.update(dx=dx.float().cpu().numpy(), dw_r=dw_r.cpu().numpy(), dgate=f.dgate.cpu().numpy(),
               **{n: v.cpu().numpy() for n, v in grads.items()})
    torch.cuda.synchronize()
    return out


def oracle_lora(orc, cfg, inp, lora, lg, ti, lb_weight=0.0):
    ref = OL.lora_backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lora, lg, ti, inp["dy"],
                           cfg.act, cfg.gate)
    ref["y"] = OL.lora_forward(inp["x"], inp["w1"], inp["w2"], lora, lg, ti, cfg.act, cfg.gate)
    if lb_weight:
        _, dl = orc.balance(lg, ti)
        ref["dx"] = ref["dx"] + lb_weight * (dl @ np.asarray(inp["w_r"], np.float64))
        ref["dw_r"] = ref["dw_r"] + lb_weight * (dl.T @ np.asarray(inp["x"], np.float64))
    return ref


def _parity(orc, cfg, T, rank=16, lb_weight=0.0, names=NAMES):
    inp = S.make_inputs(cfg, T)
    lora = S.make_lora(cfg, rank)
    got = gpu_run_lora(cfg, T, inp, lora, rank, balance_weight=lb_weight)
    assert np.array_equal(got["topk_idx"], orc.topk(got["logits"], cfg.k))
    lg = orc.router(inp["x"], inp["w_r"])
    ref = oracle_lora(orc, cfg, inp, lora, lg, got["topk_idx"], lb_weight)
    errs = {}
    for n in names:
        if n == "dw_r" and cfg.gate == S.GATE_NONE and not lb_weight:
            assert np.all(got[n] == 0), "GATE_NONE: router gets no gradient"
            continue
        errs[n] = relerr(got[n].reshape(np.shape(ref[n])), ref[n])
    bad = {n: e for n, e in errs.items() if not e <= TOL["bf16"]}
    assert not bad, f"{cfg.name} r={rank}: {errs}"
    return got, ref, errs


@pytest.mark.parametrize("name,T", [("bert", 700), ("opt", 400), ("llama", 300)])
def test_lora_configs(orc, name, T):
    _parity(orc, S.CONFIGS[name], T)


@pytest.mark.parametrize("rank", [1, 8, 32])
def test_lora_ranks(orc, rank):
    _parity(orc, S.CONFIGS["llama"], 260, rank=rank)          # SwiGLU: m' r up to 64


def test_lora_rank64_single_projection(orc):
    _parity(orc, S.CONFIGS["bert"], 300, rank=64)              # m' = 1: r = 64 fills the K stage


def test_lora_gate_none(orc):
    _parity(orc, S.CONFIGS["opt"].with_(gate=S.GATE_NONE), 257)


def test_lora_with_balance_loss(orc):
    _parity(orc, S.CONFIGS["bert"], 500, lb_weight=0.5)


@pytest.mark.parametrize("name,d,D,G,k,act", [
    ("g8k4", 512, 4096, 8, 4, S.ACT_RELU),          # the paper's G = 8, beta = 1/2 (bw 512)
    ("wide512sw", 256, 1024, 2, 1, S.ACT_SWIGLU),   # SwiGLU m' bw = 1024
    ("bw192", 256, 1536, 8, 3, S.ACT_GELU),
])
def test_lora_wide_blocks(orc, name, d, D, G, k, act):
    _parity(orc, S.FfnConfig(name, d, D, G, k, 500, "bf16", act), 500)


def test_lora_accumulate(orc):
    cfg = S.CONFIGS["bert"]
    T, rank = 300, 16
    inp = S.make_inputs(cfg, T)
    lora = S.make_lora(cfg, rank)
    base = gpu_run_lora(cfg, T, inp, lora, rank)
    rng = np.random.default_rng(0)
    prev = {n: rng.standard_normal(base[n].shape).astype(np.float32)
            for n in ("db1", "dc1", "db2", "dc2", "dw_r")}
    acc = gpu_run_lora(cfg, T, inp, lora, rank, accumulate_from=prev)
    for n, p in prev.items():
        assert relerr(acc[n], base[n] + p) < 1e-6, n


def test_lora_empty_batch():
    import torch
    import paper_2312_10365_b200 as P
    cfg = S.CONFIGS["bert"]
    f = P.RoutedLoRAFFN(0, cfg.d, cfg.D, cfg.G, cfg.k, torch.bfloat16, cfg.act, 16)
    lora = {n: to_dev(v, cfg) for n, v in S.make_lora(cfg, 16).items()}
    z = torch.empty(0, cfg.d, dtype=torch.bfloat16, device="cuda")
    w = {n: to_dev(v, cfg) for n, v in S.make_inputs(cfg, 1, need=("w1", "w2", "w_r")).items()}
    for g in f.grads.values():
        g.fill_(7.0)
    f.route(z, w["w_r"])
    f.forward(z, w["w1"], w["w2"], lora)
    _, grads, dw_r = f.backward(z, w["w1"], w["w2"], w["w_r"], lora, z)
    torch.cuda.synchronize()
    assert all(float(g.abs().max()) == 0 for g in grads.values()) and float(dw_r.abs().max()) == 0


def test_lora_deterministic(orc):
    cfg = S.CONFIGS["llama"]
    inp = S.make_inputs(cfg, 200)
    lora = S.make_lora(cfg, 16)
    a = gpu_run_lora(cfg, 200, inp, lora, 16)
    b = gpu_run_lora(cfg, 200, inp, lora, 16)
    for n in NAMES:
        assert np.array_equal(a[n], b[n]), n


# BASELINE sizes (bench.py's launch configuration), on outputs the oracle computes
# one by one: the LoRA-wrapped FFN equals the plain routed FFN on the merged
# weights W + BC (pinned in test_oracle_lora.py), so the per-token /
# per-block C oracle on merged fp64 weights gives sampled rows of y, dx, dgate and,
# through the chain rule, of dC_I and dB_O for sampled blocks.  dB_I and dC_O sum
# over every block; they are checked by the exact rescaling invariances
# <dB_I, B_I> = <dC_I, C_I> and <dB_O, B_O> = <dC_O, C_O> (y is unchanged under
# B -> sB, C -> C/s).  ReLU configs are left to the small cases: at 10^5-10^6
# pairs a few pre-activations sit within fp32 rounding of the kink.
@pytest.mark.parametrize("name,n_blocks", [("bert", 2), ("llama_scale", 1)])
def test_lora_fullsize_sampled(orc, name, n_blocks):
    cfg = S.ALL_CONFIGS[name]
    T, r = cfg.T, 16
    inp = S.make_inputs(cfg, T)
    lora = S.make_lora(cfg, r)
    got = gpu_run_lora(cfg, T, inp, lora, r)
    ti = orc.topk(got["logits"], cfg.k)
    assert np.array_equal(got["topk_idx"], ti)
    lg = orc.router(inp["x"], inp["w_r"])   # the oracle's own fp64 logits (gates), full T
    assert relerr(got["logits"], lg) <= 1e-4
    w1m, w2m = OL.merged_weights(inp["w1"], inp["w2"], lora, cfg.act)
    rng = np.random.default_rng(cfg.seed + 1)
    tokens = np.unique(np.concatenate([[0, T - 1], rng.integers(0, T, 14)])).astype(np.int64)
    blocks = np.unique(rng.integers(0, cfg.G, n_blocks)).astype(np.int32)
    tol = TOL["bf16"]
    y = orc.forward(inp["x"], w1m, w2m, lg, ti, cfg.act, cfg.gate, tokens=tokens)
    assert relerr(got["y"][tokens], y[tokens]) <= tol
    ref = orc.backward(inp["x"], w1m, w2m, inp["w_r"], lg, ti, inp["dy"], cfg.act, cfg.gate,
                       tokens=tokens, blocks=blocks)
    for n in ("dx", "dgate"):
        assert relerr(got[n][tokens], ref[n][tokens]) <= tol, n
    assert relerr(got["dw_r"][blocks], ref["dw_r"][blocks]) <= tol
    mp, bw = cfg.mprime, cfg.bw
    rows = np.concatenate([np.arange(b * bw, (b + 1) * bw) for b in blocks])
    dw1 = ref["dw1"].reshape((mp,) + ref["dw1"].shape[-2:])
    b1 = np.asarray(lora["b1"], np.float64).reshape(mp, r, cfg.d)
    gc1 = got["dc1"].reshape(mp, cfg.D, r)
    for m in range(mp):  # w1' = w1 + c1 b1  =>  dc1 = dw1' b1^T
        assert relerr(gc1[m][rows], dw1[m][rows] @ b1[m].T) <= tol
    assert relerr(got["db2"][rows], ref["dw2"][rows] @ np.asarray(lora["c2"], np.float64).T) <= tol

    def dot(a, b):
        return float(np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)))

    for (ga, fa), (gb, fb) in [(("db1", "b1"), ("dc1", "c1")), (("db2", "b2"), ("dc2", "c2"))]:
        lhs = dot(got[ga], np.asarray(lora[fa]).reshape(got[ga].shape))
        rhs = dot(got[gb], np.asarray(lora[fb]).reshape(got[gb].shape))
        scale = np.sqrt(dot(got[ga], got[ga]) * dot(lora[fa], lora[fa]))
        assert abs(lhs - rhs) <= tol * scale, (ga, gb, lhs, rhs)

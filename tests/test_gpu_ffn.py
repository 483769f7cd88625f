"""GPU parity of the routed-FFN forward and backward against the fp64 oracle.

Inputs: synthetic seeded tensors (synthetic/).  Routing: either the GPU's own
router (then the oracle is given the same top-k, which test_gpu_route checks
bit-exactly) or fixed generator logits via SPT_ROUTE_LOGITS_IN.  Error metric:
infinity-norm relative error (reading c14), bound 1e-4 fp32 / 2e-2 bf16
(BASELINE.json north_star).  Sizes span several 128-row tiles and ragged
tails; full BASELINE sizes are covered by sampled rows/blocks in
test_gpu_fullsize.py.
"""
import numpy as np
import pytest

import synthetic as S
from helpers import TOL, gpu_run, oracle_run, relerr, relu_kink_fixup

pytestmark = pytest.mark.gpu

NAMES = ("y", "dx", "dw1", "dw2", "dw_r", "dgate")


def _check(cfg, got, ref, names=NAMES, tol=None):
    tol = TOL[cfg.dtype] if tol is None else tol
    errs = {}
    for n in names:
        if n == "dw_r" and cfg.gate == S.GATE_NONE:
            assert np.all(got[n] == 0), "GATE_NONE: router gets no gradient"
            continue
        errs[n] = relerr(got[n], ref[n])
    bad = {n: e for n, e in errs.items() if not e <= tol}
    assert not bad, f"{cfg.name}: {errs}"
    return errs


def _parity(orc, cfg, T, kind=None, names=NAMES):
    inp = S.make_inputs(cfg, T)
    logits = None if kind is None else S.make_logits(T, cfg.G, cfg.k, kind, seed=cfg.seed)
    got = gpu_run(cfg, T, inp, logits_in=logits)
    lg = logits.astype(np.float64) if logits is not None else orc.router(inp["x"], inp["w_r"])
    # the GPU's selection (checked bit-exact against the oracle's top-k in test_gpu_route)
    assert np.array_equal(got["topk_idx"], orc.topk(got["logits"], cfg.k))
    ref = oracle_run(orc, cfg, inp, lg, got["topk_idx"])
    if cfg.dtype == "f32":  # fp32 bound: ReLU kink decisions taken in each side's precision
        relu_kink_fixup(cfg, inp, lg, got["topk_idx"], got, ref)
    return _check(cfg, got, ref, names)


@pytest.mark.parametrize("gate", [S.GATE_SIGMOID, S.GATE_NONE])
@pytest.mark.parametrize("T", [256, 1, 131, 1000])
def test_tiny_fp32(orc, T, gate):
    _parity(orc, S.CONFIGS["tiny"].with_(gate=gate), T)


@pytest.mark.parametrize("kind", ["normal", "zipf", "same", "ties"])
def test_tiny_fixed_logits(orc, kind):
    _parity(orc, S.CONFIGS["tiny"], 700, kind=kind)


@pytest.mark.parametrize("act", [S.ACT_RELU, S.ACT_GELU, S.ACT_SWIGLU])
def test_fp32_all_activations(orc, act):
    cfg = S.CONFIGS["tiny"].with_(act=act, name=f"tiny-act{act}")
    _parity(orc, cfg, 333)


@pytest.mark.parametrize("name,T", [("bert", 1000), ("opt", 600), ("llama", 300)])
def test_bf16_configs(orc, name, T):
    _parity(orc, S.CONFIGS[name], T)


@pytest.mark.parametrize("name", ["bert", "opt", "llama"])
def test_bf16_gate_none(orc, name):
    _parity(orc, S.CONFIGS[name].with_(gate=S.GATE_NONE), 257)


@pytest.mark.parametrize("kind", ["zipf", "same"])
def test_bf16_skewed_buckets(orc, kind):
    """Skewed / degenerate bucket sizes: empty buckets and k buckets of size T."""
    _parity(orc, S.CONFIGS["opt"], 700, kind=kind)


def test_k_equals_G_is_dense(orc):
    cfg = S.FfnConfig("kG", 128, 512, 4, 4, 300, "bf16", S.ACT_SWIGLU)
    _parity(orc, cfg, 300)


@pytest.mark.parametrize("name,d,D,G,k,act", [("bw256", 512, 2048, 8, 2, S.ACT_GELU),
                                               ("bw192", 256, 1536, 8, 3, S.ACT_RELU)])
def test_wide_blocks(orc, name, d, D, G, k, act):
    """128 < m'*bw <= 256 with m' = 1: FWD1 and dA both take the CTA-pair gather
    kernel (N > 128), B split into halves of bw/2 rows per CTA."""
    _parity(orc, S.FfnConfig(name, d, D, G, k, 700, "bf16", act), 700)


@pytest.mark.parametrize("name,d,D,G,k,act", [
    ("wide1024", 256, 2048, 2, 1, S.ACT_GELU),      # bw 1024: 4 FWD1 / 8 dA unit tiles
    ("wide512sw", 256, 1024, 2, 1, S.ACT_SWIGLU),   # bw 512 SwiGLU: m' bw = 1024
    ("wide1376", 256, 2752, 2, 1, S.ACT_GELU),      # bw 1376: partial unit / feature tiles
    ("g8k4", 512, 4096, 8, 4, S.ACT_RELU),          # the paper's G = 8, beta = 1/2 shape
])
def test_wide_blocks_tiled(orc, name, d, D, G, k, act):
    """m' bw > 256 (the paper's G = 4 / 8 blocks): FWD1 / dA tile
    the block's units (dA's dgate summed over the unit tiles by dgate_reduce),
    FWD2 / dX stream K, dW1 / dW2 tile the features."""
    _parity(orc, S.FfnConfig(name, d, D, G, k, 600, "bf16", act), 600)


@pytest.mark.parametrize("name", ["opt2048_g8_b34", "llama4096_g8_b34", "opt2048_g4", "llama4096_g4",
                                  "opt2048_g4_b34", "llama4096_g4_b34"])
def test_paper_g4_g8_beta(orc, name):
    """the paper's G = 4 / 8 groups at beta = 1/2 and 3/4 (Table 5,
    PAPER.md:1023-1026, 1043-1046; "G (e.g., 4 or 8)"), full shapes
    (bw 1024-2752) at a T the oracle's full backward covers in seconds."""
    _parity(orc, S.PAPER_CONFIGS[name], 300)


@pytest.mark.parametrize("name", ["opt2048_g8_f32", "llama4096_g8_f32", "opt2048_g8_b34_f32",
                                  "llama4096_g8_b34_f32"])
def test_paper_fp32(orc, name):
    """SURVEY §8(f) f1 at the paper's own precision (fp32; Table 5):
    fp32 tensors on the bf16 tensor cores as hi + lo halves (three products per
    GEMM, reading c13'), held to the fp32 bound 1e-4 at the full G = 8 shapes."""
    _parity(orc, S.PAPER_CONFIGS[name], 300)


@pytest.mark.parametrize("name,T", [("bert", 600), ("opt", 300), ("llama", 257)])
def test_fp32_tensor_core_shapes(orc, name, T):
    """The split fp32 path at the BASELINE block shapes (bw 96 / 128, GELU, ReLU,
    SwiGLU; K streamed in three passes for FWD2 / dX) against the 1e-4 bound."""
    _parity(orc, S.CONFIGS[name].with_(dtype="f32", name=f"{name}-f32"), T)


@pytest.mark.parametrize("G,k", [(129, 8), (256, 16)])
def test_bf16_many_blocks(orc, G, k):
    """Reading c25: G in 129..256 on the tcgen05 path (router N = 144 / 256, dW_R
    as two 128-block M halves), bit-exact routing and the bf16 bound."""
    _parity(orc, S.FfnConfig(f"G{G}", 256, G * 64, G, k, 900, "bf16", S.ACT_GELU), 900)


def test_k1_bf16(orc):
    cfg = S.FfnConfig("k1", 256, 2048, 16, 1, 400, "bf16", S.ACT_GELU)
    _parity(orc, cfg, 400)


def test_empty_batch():
    import torch
    import paper_2312_10365_b200 as P
    f = P.RoutedFFN(0, 128, 512, 8, 2, torch.float32, P.SPT_ACT_RELU)
    x = torch.empty(0, 128, device="cuda")
    w1 = torch.randn(512, 128, device="cuda")
    w2 = torch.randn(512, 128, device="cuda")
    w_r = torch.randn(8, 128, device="cuda")
    f.route(x, w_r)
    f.forward(x, w1, w2)
    f.dw1.fill_(7)
    f.backward(x, w1, w2, w_r, x)
    torch.cuda.synchronize()
    assert f.route_buf.block_offsets.cpu().tolist() == [0] * 9
    assert float(f.dw1.abs().max()) == 0.0


def test_empty_batch_bf16():
    """T = 0 on the tcgen05 path (LLaMA shapes): no launch reads a token, the
    buckets are empty and dW are zeroed (SPT_BWD_ACCUMULATE_DW off)."""
    import torch
    import paper_2312_10365_b200 as P
    cfg = S.CONFIGS["llama"]
    f = P.RoutedFFN(0, cfg.d, cfg.D, cfg.G, cfg.k, torch.bfloat16, cfg.act)
    x = torch.empty(0, cfg.d, device="cuda", dtype=torch.bfloat16)
    w1 = torch.randn(2, cfg.D, cfg.d, device="cuda").to(torch.bfloat16)
    w2 = torch.randn(cfg.D, cfg.d, device="cuda").to(torch.bfloat16)
    w_r = torch.randn(cfg.G, cfg.d, device="cuda").to(torch.bfloat16)
    f.route(x, w_r)
    f.forward(x, w1, w2)
    f.dw1.fill_(7)
    f.dw_r.fill_(7)
    f.backward(x, w1, w2, w_r, x)
    torch.cuda.synchronize()
    assert f.route_buf.block_offsets.cpu().tolist() == [0] * (cfg.G + 1)
    assert float(f.dw1.abs().max()) == 0.0 and float(f.dw_r.abs().max()) == 0.0


@pytest.mark.parametrize("name", ["bert", "llama"])
def test_single_token_bf16(orc, name):
    """T = 1: every selected block holds one row of a 128-row tile (ragged in
    every bucket), the other G - k buckets are empty."""
    _parity(orc, S.CONFIGS[name], 1)


@pytest.mark.parametrize("name", ["tiny", "bert"])
def test_accumulate_dw(orc, name):
    cfg = S.CONFIGS[name]
    T = 300
    inp = S.make_inputs(cfg, T)
    base = gpu_run(cfg, T, inp)
    rng = np.random.default_rng(0)
    prior = {n: rng.standard_normal(base[n].shape).astype(np.float32) for n in ("dw1", "dw2", "dw_r")}
    acc = gpu_run(cfg, T, inp, accumulate_from=prior)
    for n in ("dw1", "dw2", "dw_r"):
        assert relerr(acc[n] - prior[n], base[n]) < 1e-5


@pytest.mark.parametrize("name", ["tiny", "bert", "llama"])
def test_deterministic(orc, name):
    """Bitwise-reproducible results run to run (ascending-block k-way sums,
    reading c12), with and without the SPT_FFN_DETERMINISTIC bit, which every
    path already honours (include/spt_ffn.h)."""
    cfg = S.CONFIGS[name]
    T = 513
    inp = S.make_inputs(cfg, T)
    a = gpu_run(cfg, T, inp)
    b = gpu_run(cfg, T, inp)
    c = gpu_run(cfg, T, inp, deterministic=True)
    for n in NAMES + ("logits", "bucket_token"):
        assert np.array_equal(a[n], b[n]), n
        assert np.array_equal(a[n], c[n]), n


def test_ragged_tail_multi_tile(orc):
    """T = 5000 BERT tokens: several 128-row tiles per block and a ragged last
    tile in every bucket."""
    _parity(orc, S.CONFIGS["bert"], 5000)


@pytest.mark.parametrize("kind", ["zipf", "same"])
def test_deterministic_path_skewed(orc, kind):
    """The deterministic (partial rows + ordered combine) path keeps its parity
    coverage on skewed buckets too."""
    cfg = S.CONFIGS["llama"]
    T = 700
    inp = S.make_inputs(cfg, T)
    logits = S.make_logits(T, cfg.G, cfg.k, kind, seed=cfg.seed)
    got = gpu_run(cfg, T, inp, logits_in=logits, deterministic=True)
    ref = oracle_run(orc, cfg, inp, logits.astype(np.float64), got["topk_idx"])
    _check(cfg, got, ref)


@pytest.mark.parametrize("name", ["tiny", "llama"])
def test_dw_event_marks_final_gradients(orc, name):
    """spt_ffn_backward records dw_event once dw1/dw2/dw_r are final (before dx):
    snapshots taken on another stream right after the event equal the results."""
    import torch
    import paper_2312_10365_b200 as P
    from helpers import to_dev, torch_dtype
    cfg = S.CONFIGS[name]
    T = 700
    inp = S.make_inputs(cfg, T)
    f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, torch_dtype(cfg), cfg.act, cfg.gate)
    x, w1, w2, w_r, dy = (to_dev(inp[n], cfg) for n in ("x", "w1", "w2", "w_r", "dy"))
    f.route(x, w_r)
    f.forward(x, w1, w2)
    ev = torch.cuda.Event()
    f.backward(x, w1, w2, w_r, dy, dw_event=ev)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        side.wait_event(ev)
        snap = [t.clone() for t in (f.dw1, f.dw2, f.dw_r)]
    torch.cuda.synchronize()
    for a, b in zip(snap, (f.dw1, f.dw2, f.dw_r)):
        assert torch.equal(a, b)

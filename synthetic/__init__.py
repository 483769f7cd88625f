"""Seeded synthetic inputs for the SPT routed FFN (arXiv 2312.10365).

This module is shared by the CUDA path's tests/bench AND by the CPU oracle's
tests.  It holds NO arithmetic of the method (no routing, no GEMM, no
activation): only the workload shapes and seeded random draws.

Workload recipe:
  * The paper's micro-benchmarks use "Random", "randomly generated sequences"
    (§6.1) for every block-level experiment; the
    FFN treats batch x sequence as a flat token batch (§6.2).
  * Shapes come from BASELINE.json ``configs``.
  * One seed per config, ``20231216 + cfg_index``; every tensor draws from its
    own PCG64 stream ``SeedSequence([seed, tensor_id])`` in fp64 and is then
    rounded ONCE, round-to-nearest-even, to the storage dtype (fp32 or bf16).
    The identical bits go to the GPU and to the oracle.
  * x ~ N(0,1); w1 ~ N(0,1/d) (so z ~ N(0,1)); w2 ~ N(0, 1/(k*bw));
    w_r ~ N(0,1/d) (so logits ~ N(0,1)); dy ~ N(0,1).
  * Fixed-logit variants (routing parity):
    "normal" N(0,1) fp32, "zipf" (per-block Zipf bias -> skewed bucket sizes),
    "same" (every token picks blocks 0..k-1: k buckets of size T, rest empty),
    "ties" (small integers -> massive exact ties, incl. +0/-0).

Arrays are returned as numpy float32 holding values exactly representable in
the requested dtype ("bf16" values have at most 8 significant bits).
"""
from __future__ import annotations

import dataclasses
import numpy as np

ACT_RELU, ACT_GELU, ACT_SWIGLU = 0, 1, 2
GATE_SIGMOID, GATE_NONE = 0, 1
ACT_NAMES = {"relu": ACT_RELU, "gelu": ACT_GELU, "swiglu": ACT_SWIGLU}
GATE_NAMES = {"sigmoid": GATE_SIGMOID, "none": GATE_NONE}

BASE_SEED = 20231216


@dataclasses.dataclass(frozen=True)
class FfnConfig:
    """One routed-FFN workload.  Field names follow SURVEY.md §8 notation."""
    name: str
    d: int          # d_model (X in R^{n x d})
    D: int          # d_ff, intermediate dim of W_I in R^{d x D}
    G: int          # number of blocks
    k: int          # activated blocks per token, G'
    T: int          # tokens = batch * seq
    dtype: str      # "f32" | "bf16" storage dtype
    act: int        # ACT_*
    gate: int = GATE_SIGMOID
    cfg_index: int = 0

    @property
    def bw(self) -> int:
        return self.D // self.G

    @property
    def mprime(self) -> int:
        return 2 if self.act == ACT_SWIGLU else 1

    @property
    def seed(self) -> int:
        return BASE_SEED + self.cfg_index

    def with_(self, **kw) -> "FfnConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": FfnConfig("tiny", 128, 512, 8, 2, 256, "f32", ACT_RELU, cfg_index=0),
    "bert": FfnConfig("bert", 768, 3072, 32, 8, 16 * 512, "bf16", ACT_GELU, cfg_index=1),
    "opt": FfnConfig("opt", 2048, 8192, 64, 16, 8 * 1024, "bf16", ACT_RELU, cfg_index=2),
    "llama": FfnConfig("llama", 4096, 11008, 86, 22, 8 * 2048, "bf16", ACT_SWIGLU, cfg_index=3),
    # scaling run: 8 x 4096 tokens per GPU (weak scaling)
    "llama_scale": FfnConfig("llama_scale", 4096, 11008, 86, 22, 8 * 4096, "bf16", ACT_SWIGLU,
                             cfg_index=4),
}

# the paper's own FFN workload (Table 5, PAPER.md:1011-1048;
# Table 3 shapes): OPT-2048 / LLaMA-4096 2-matrix FFNs, batch
# 16 x 512 tokens, G = 8 blocks, beta = k/G = 1/2.  The
# paper's LLaMA-family block uses GELU in its 2-matrix form.
# Table 5 also times beta = 3/4 ("SPT (3/4)"), and the router
# section names G = 4 as the other default group count ("a small G (e.g., 4 or
# 8)"): k = beta * G gives k = 6 of 8, k = 2 of 4 and k = 3 of 4.
PAPER_CONFIGS = {
    "opt2048_g8": FfnConfig("opt2048_g8", 2048, 8192, 8, 4, 16 * 512, "bf16", ACT_RELU, cfg_index=5),
    "llama4096_g8": FfnConfig("llama4096_g8", 4096, 11008, 8, 4, 16 * 512, "bf16", ACT_GELU,
                              cfg_index=6),
    "opt2048_g8_b34": FfnConfig("opt2048_g8_b34", 2048, 8192, 8, 6, 16 * 512, "bf16", ACT_RELU,
                                cfg_index=7),
    "llama4096_g8_b34": FfnConfig("llama4096_g8_b34", 4096, 11008, 8, 6, 16 * 512, "bf16", ACT_GELU,
                                  cfg_index=8),
    "opt2048_g4": FfnConfig("opt2048_g4", 2048, 8192, 4, 2, 16 * 512, "bf16", ACT_RELU, cfg_index=9),
    "llama4096_g4": FfnConfig("llama4096_g4", 4096, 11008, 4, 2, 16 * 512, "bf16", ACT_GELU,
                              cfg_index=20),
    "opt2048_g4_b34": FfnConfig("opt2048_g4_b34", 2048, 8192, 4, 3, 16 * 512, "bf16", ACT_RELU,
                                cfg_index=21),
    "llama4096_g4_b34": FfnConfig("llama4096_g4_b34", 4096, 11008, 4, 3, 16 * 512, "bf16", ACT_GELU,
                                  cfg_index=22),
    # Table 5's own precision: fp32 ("single-precision") at beta = 1/2
    # and 3/4, G = 8 -- the configurations the paper quotes 54.9 / 84.6 ms (OPT-2048)
    # and 150.8 / 228.9 ms (LLaMA-4096) for
    "opt2048_g8_f32": FfnConfig("opt2048_g8_f32", 2048, 8192, 8, 4, 16 * 512, "f32", ACT_RELU,
                                cfg_index=23),
    "llama4096_g8_f32": FfnConfig("llama4096_g8_f32", 4096, 11008, 8, 4, 16 * 512, "f32", ACT_GELU,
                                  cfg_index=24),
    "opt2048_g8_b34_f32": FfnConfig("opt2048_g8_b34_f32", 2048, 8192, 8, 6, 16 * 512, "f32",
                                    ACT_RELU, cfg_index=25),
    "llama4096_g8_b34_f32": FfnConfig("llama4096_g8_b34_f32", 4096, 11008, 8, 6, 16 * 512, "f32",
                                      ACT_GELU, cfg_index=26),
}
ALL_CONFIGS = {**CONFIGS, **PAPER_CONFIGS}

_TENSOR_IDS = {"x": 1, "w1": 2, "w2": 3, "w_r": 4, "dy": 5, "logits": 6,
               "b1": 7, "c1": 8, "b2": 9, "c2": 10, "pq": 11}


def _stream(seed: int, name: str, extra: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _TENSOR_IDS[name], extra])))


def round_to_dtype(a: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp64 values once (RNE) to fp32 or bf16; return float32 array."""
    a = np.asarray(a, dtype=np.float64)
    if dtype == "f32":
        return a.astype(np.float32)
    if dtype == "bf16":
        m, e = np.frexp(a)                      # a = m * 2^e, 0.5 <= |m| < 1
        m = np.rint(np.ldexp(m, 8))             # 8 significant bits, ties-to-even
        return np.ldexp(m, e - 8).astype(np.float32)
    raise ValueError(dtype)


def bf16_bits(a32: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns of float32 values already exact in bf16."""
    u = np.ascontiguousarray(a32, dtype=np.float32).view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "value not exactly representable in bf16"
    return (u >> 16).astype(np.uint16)


def make_inputs(cfg: FfnConfig, T: int | None = None, need=("x", "w1", "w2", "w_r", "dy"),
                token_offset: int = 0) -> dict:
    """Seeded inputs for ``cfg`` (optionally overriding the token count T).

    x, dy: [T, d]; w1: [D, d] (or [2, D, d] for SwiGLU: gate, up) = W_I^T of
    Eq. 4; w2: [D, d] = W_O; w_r: [G, d] = W_R^T.
    Token rows are drawn independently per token index, so the first T' rows of a
    T-token draw equal a T'-token draw (used for sampled oracle checks), and
    ``token_offset`` (a multiple of 1024) selects rows [offset, offset+T) of the
    global token stream (data-parallel shards: weights identical, tokens disjoint).
    """
    T = cfg.T if T is None else T
    s, d, D, G, k, bw, dt = cfg.seed, cfg.d, cfg.D, cfg.G, cfg.k, cfg.bw, cfg.dtype
    out = {}
    if "x" in need:
        out["x"] = _token_rows(s, "x", T, d, 1.0, dt, token_offset)
    if "dy" in need:
        out["dy"] = _token_rows(s, "dy", T, d, 1.0, dt, token_offset)
    if "w1" in need:
        shape = (2, D, d) if cfg.act == ACT_SWIGLU else (D, d)
        out["w1"] = round_to_dtype(_stream(s, "w1").standard_normal(shape) / np.sqrt(d), dt)
    if "w2" in need:
        out["w2"] = round_to_dtype(_stream(s, "w2").standard_normal((D, d)) / np.sqrt(k * bw), dt)
    if "w_r" in need:
        out["w_r"] = round_to_dtype(_stream(s, "w_r").standard_normal((G, d)) / np.sqrt(d), dt)
    return out


LORA_RANK = 16  # d_lora default


def make_lora(cfg: FfnConfig, r: int = LORA_RANK) -> dict:
    """Seeded LoRA factors of both FFN projections (PAPER.md:159
    Y = XW + XBC, B in R^{d x r}, C in R^{r x h}), in the library's storage:
      b1 = B_I^T [m', r, d], c1 = C_I^T [m', D, r], b2 = B_O [D, r], c2 = C_O [r, d]
    (m' = 2 for SwiGLU: gate, up; the leading axis is dropped for m' = 1).
    Scales: b1 ~ N(0, 1/d) (u = x B_I ~ N(0,1)); c1 ~ N(0, 0.25/r) (the LoRA term of
    z ~ N(0, 1/4), next to x W_I ~ N(0,1)); b2 ~ N(0, 1/(k bw)); c2 ~ N(0, 0.25/r).
    Both factors are non-zero (LoRA's usual zero init of one factor would make
    the other's gradient vanish and the parity check vacuous)."""
    s, d, D, k, bw, dt = cfg.seed, cfg.d, cfg.D, cfg.k, cfg.bw, cfg.dtype
    mp = cfg.mprime
    lead = (mp,) if mp == 2 else ()
    c = np.sqrt(0.25 / r)
    return {
        "b1": round_to_dtype(_stream(s, "b1", r).standard_normal(lead + (r, d)) / np.sqrt(d), dt),
        "c1": round_to_dtype(_stream(s, "c1", r).standard_normal(lead + (D, r)) * c, dt),
        "b2": round_to_dtype(_stream(s, "b2", r).standard_normal((D, r)) / np.sqrt(k * bw), dt),
        "c2": round_to_dtype(_stream(s, "c2", r).standard_normal((r, d)) * c, dt),
    }


# sparse-MHA top-L selection (Alg. 3) on PQ codes.  The paper's
# PQ: codeword dimension d' = 8 and E = 16 codewords per codebook,
# so M = head_dim / 8 codebooks (8 for 64-dim heads: BERT-base, OPT-1.3B; 16 for
# LLaMA-7B's 128-dim heads); L = lambda n with lambda = 1/8 (the
# paper's "top-L as lambda n").
@dataclasses.dataclass(frozen=True)
class ToplConfig:
    name: str
    heads: int      # batch x heads: independent (sequence, head) problems
    n: int          # sequence length (queries = keys)
    M: int          # codebooks
    E: int = 16     # codewords per codebook
    lam: float = 0.125
    causal: bool = False
    cfg_index: int = 10

    @property
    def L(self) -> int:
        return max(1, int(self.lam * self.n))

    @property
    def seed(self) -> int:
        return BASE_SEED + self.cfg_index

    def with_(self, **kw) -> "ToplConfig":
        return dataclasses.replace(self, **kw)


TOPL_CONFIGS = {
    "topl_tiny": ToplConfig("topl_tiny", 2, 256, 8, cfg_index=10),
    "topl_bert": ToplConfig("topl_bert", 16 * 12, 512, 8, cfg_index=11),      # batch 16, 12 heads
    "topl_opt": ToplConfig("topl_opt", 8 * 32, 1024, 8, causal=True, cfg_index=12),
    "topl_llama": ToplConfig("topl_llama", 8 * 32, 2048, 16, causal=True, cfg_index=13),
}


def make_pq_codes(cfg: "ToplConfig", heads: int | None = None) -> tuple:
    """Seeded PQ code matrices (queries, keys) [heads, n, M] uint8 in [0, E).

    Real queries / keys are clustered (that is why PQ finds the top-L, PAPER.md:
    306), so codes are drawn around per-head cluster templates: each token picks
    one of 8 templates and keeps each codebook's template codeword with
    probability 0.6, else draws it uniformly -- indicator scores then span 0..M
    with many ties (the integer-ranking regime of Eq. 3).  No arithmetic of the
    method is done here (no quantisation, no scoring)."""
    H = cfg.heads if heads is None else heads
    g = _stream(cfg.seed, "pq", H)
    tmpl = g.integers(0, cfg.E, size=(H, 8, cfg.M))
    out = []
    for _ in range(2):
        pick = g.integers(0, 8, size=(H, cfg.n))
        base = np.take_along_axis(tmpl, pick[:, :, None].repeat(cfg.M, axis=2), axis=1)
        keep = g.random((H, cfg.n, cfg.M)) < 0.6
        codes = np.where(keep, base, g.integers(0, cfg.E, size=(H, cfg.n, cfg.M)))
        out.append(codes.astype(np.uint8))
    return out[0], out[1]


_ROW_CHUNK = 1024


def _token_rows(seed, name, T, d, std, dtype, offset=0):
    """[T, d] rows drawn in chunks of 1024 tokens, each chunk its own stream, so
    that any prefix (and any chunk) can be regenerated without the whole tensor."""
    if offset % _ROW_CHUNK:
        raise ValueError("token_offset must be a multiple of 1024")
    out = np.empty((T, d), dtype=np.float32)
    for c0 in range(0, T, _ROW_CHUNK):
        c1 = min(T, c0 + _ROW_CHUNK)
        g = _stream(seed, name, 1 + (offset + c0) // _ROW_CHUNK)
        out[c0:c1] = round_to_dtype(g.standard_normal((_ROW_CHUNK, d))[: c1 - c0] * std, dtype)
    return out


def make_logits(T: int, G: int, k: int, kind: str = "normal", seed: int = BASE_SEED) -> np.ndarray:
    """Fixed fp32 router logits [T, G] for routing parity (fed to both sides)."""
    g = _stream(seed, "logits", {"normal": 0, "zipf": 1, "same": 2, "ties": 3, "signed0": 4}[kind])
    if kind == "normal":
        a = g.standard_normal((T, G))
    elif kind == "zipf":
        bias = 3.0 / (1.0 + np.arange(G)) ** 1.1          # block 0 most popular
        a = g.standard_normal((T, G)) * 0.5 + bias[None, :] * np.where(g.random((T, G)) < 0.5, 1, -1)
    elif kind == "same":
        a = g.standard_normal((T, G)) * 0.1
        a[:, :k] += 10.0 * np.where(g.random((T, k)) < 0.5, 1, -1)
    elif kind == "ties":
        a = g.integers(-2, 3, size=(T, G)).astype(np.float64)
    elif kind == "signed0":
        a = np.where(g.random((T, G)) < 0.5, 0.0, -0.0) * np.ones((T, G))
        a[:, ::3] = g.integers(-1, 2, size=a[:, ::3].shape)
    else:
        raise ValueError(kind)
    return a.astype(np.float32)

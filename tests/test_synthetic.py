"""The seeded input generator: determinism, prefix property, RNE rounding."""
import numpy as np
import torch

import synthetic as S


def test_bf16_rounding_is_nearest_even():
    rng = np.random.default_rng(1)
    a = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 6, 20000),
                        [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 0.0, -0.0]])
    r = S.round_to_dtype(a, "bf16").astype(np.float64)
    S.bf16_bits(r.astype(np.float32))                   # exact in bf16
    # nearest: no bf16 value strictly closer (check both neighbours)
    b16 = S.bf16_bits(r.astype(np.float32)).astype(np.uint32)
    up = ((b16 + 1) << 16).view(np.float32).astype(np.float64)
    dn = ((b16 - 1) << 16).view(np.float32).astype(np.float64)
    err = np.abs(a - r)
    nz = r != 0
    assert np.all(err[nz] <= np.abs(a - up)[nz]) and np.all(err[nz] <= np.abs(a - dn)[nz])
    # ties to even: 1 + 2^-8 is halfway between 1 and 1+2^-7 -> 1 (even)
    assert r[-5] == 1.0 and r[-4] == 1 + 4 * 2 ** -8 and r[-3] == -1.0
    # agrees with torch's fp32 -> bf16 conversion on fp32-exact inputs
    a32 = rng.standard_normal(5000).astype(np.float32)
    t = torch.from_numpy(a32).to(torch.bfloat16).float().numpy()
    assert np.array_equal(S.round_to_dtype(a32.astype(np.float64), "bf16"), t)


def test_inputs_deterministic_and_prefix_stable():
    cfg = S.CONFIGS["bert"]
    a = S.make_inputs(cfg, T=2100)
    b = S.make_inputs(cfg, T=3000)
    assert np.array_equal(a["x"], b["x"][:2100]) and np.array_equal(a["dy"], b["dy"][:2100])
    assert np.array_equal(a["w1"], b["w1"])
    assert a["w1"].shape == (cfg.D, cfg.d) and a["w_r"].shape == (cfg.G, cfg.d)
    c = S.make_inputs(S.CONFIGS["llama"].with_(d=64, D=86 * 16), T=5)
    assert c["w1"].shape == (2, 86 * 16, 64)


def test_config_table():
    c = S.CONFIGS
    assert (c["tiny"].bw, c["bert"].bw, c["opt"].bw, c["llama"].bw) == (64, 96, 128, 128)
    assert c["llama"].T == 16384 and c["llama_scale"].T == 32768
    assert all(cfg.D % cfg.G == 0 for cfg in c.values())

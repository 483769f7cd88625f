"""Diagnostic (tool): where does fp32 dx differ from the oracle after the ReLU kink fix-up?"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import oracle as orc
import synthetic as S
from helpers import gpu_run, oracle_run, relu_kink_fixup

cfg = S.PAPER_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "opt2048_g8_b34_f32"]
T = 300
inp = S.make_inputs(cfg, T)
got = gpu_run(cfg, T, inp)
lg = orc.router(inp["x"], inp["w_r"])
ref = oracle_run(orc, cfg, inp, lg, got["topk_idx"])
n = relu_kink_fixup(cfg, inp, lg, got["topk_idx"], got, ref)
print("ambiguous", n)
err = np.abs(got["dx"] - ref["dx"]).max(1) / np.abs(ref["dx"]).max()
t = int(np.argmax(err))
print("worst token", t, err[t], "next", np.sort(err)[-5:])
x = inp["x"].astype(np.float64); w1 = inp["w1"].astype(np.float64); w2 = inp["w2"].astype(np.float64)
dy = inp["dy"].astype(np.float64)
r = got["dx"][t] - ref["dx"][t]
cs = []
for j in range(cfg.k):
    b = int(got["topk_idx"][t, j]); rows = slice(b * cfg.bw, (b + 1) * cfg.bw)
    z = w1[rows] @ x[t]
    da = w2[rows] @ dy[t]
    g = 1 / (1 + np.exp(-lg[t, b]))
    c = (w1[rows] @ r) / np.sum(w1[rows] ** 2, 1)
    for u in np.argsort(-np.abs(c))[:3]:
        cs.append((abs(float(c[u])), b, int(u), float(c[u]), float(z[u]), float(g * da[u])))
for e in sorted(cs, reverse=True)[:8]:
    print(" block %d unit %d: dZ diff %.4g  z %.4g  g dA %.4g" % e[1:])
print("residual norm", np.linalg.norm(r), "ref norm", np.linalg.norm(ref["dx"][t]))
print("bucket position of token in its blocks:", [int(np.nonzero((got["bucket_token"] == t))[0][j]) for j in range(cfg.k)], got["block_offsets"])

"""Diagnostic: FWD1 stash (Z, H) of a wide-block config against numpy, per pair.

usage: python tools/diag_wide.py d D G k act T   (bf16; act 0 relu, 1 gelu, 2 swiglu)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthetic as S
import paper_2312_10365_b200 as P

d, D, G, k, act, T = (int(v) for v in sys.argv[1:7])
cfg = S.FfnConfig("diag", d, D, G, k, T, "bf16", act)
inp = S.make_inputs(cfg, T)
f = P.RoutedFFN(T, d, D, G, k, torch.bfloat16, act, cfg.gate)
dev = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()
x, w1, w2, w_r = (dev(inp[n]) for n in ("x", "w1", "w2", "w_r"))
f.route(x, w_r)
f.forward(x, w1, w2)
torch.cuda.synchronize()
rb = f.route_buf
ti = rb.topk_idx.cpu().numpy()
ps = rb.pair_slot.cpu().numpy().reshape(T, k)
bo = rb.block_offsets.cpu().numpy()
to = rb.tile_offsets.cpu().numpy()
bw, mp = D // G, cfg.mprime
rows_cap = T * k + 128 * G
stash = f.stash.view(torch.bfloat16)
z = stash[: rows_cap * mp * bw].view(rows_cap, mp * bw).float().cpu().numpy()
zbytes = (rows_cap * mp * bw * 2 + 255) // 256 * 256
h = stash[zbytes // 2: zbytes // 2 + rows_cap * bw].view(rows_cap, bw).float().cpu().numpy()
xf = x.float().cpu().numpy()
w1f = w1.float().cpu().numpy().reshape(mp * D, d)
print("tile_offsets", to, "block_offsets", bo)
for t in range(min(T, 3)):
    for j in range(k):
        b = ti[t, j]
        prow = to[b] * 128 + (ps[t, j] - bo[b])
        zr = xf[t] @ w1f[b * bw:(b + 1) * bw].T
        if mp == 2:
            zr = np.concatenate([zr, xf[t] @ w1f[D + b * bw: D + (b + 1) * bw].T])
        err = np.abs(z[prow] - zr) / (np.abs(zr).max() + 1e-9)
        bad = np.nonzero(err > 0.02)[0]
        print(f"t={t} b={b} prow={prow} z maxerr {err.max():.3f} bad units {bad[:8]}..{bad[-4:] if len(bad) else ''} n_bad={len(bad)}")
        print("   z[:4]", z[prow, :4], "ref", zr[:4], " h[:4]", h[prow, :4])

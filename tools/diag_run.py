"""Diagnostic: time GPU route/fwd/bwd and the oracle separately for one config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import synthetic as S
from helpers import gpu_run, oracle_run, relerr
name, T = sys.argv[1], int(sys.argv[2])
skip_oracle = len(sys.argv) > 3
cfg = S.CONFIGS[name]
inp = S.make_inputs(cfg, T)
t0 = time.time()
import paper_2312_10365_b200 as P
f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, torch.float32 if cfg.dtype == "f32" else torch.bfloat16, cfg.act, cfg.gate)
dev = lambda a: torch.from_numpy(a).to(f.dtype).cuda()
x, w1, w2, w_r, dy = (dev(inp[n]) for n in ("x", "w1", "w2", "w_r", "dy"))
for stage in ("route", "forward", "backward"):
    t = time.time()
    if stage == "route": f.route(x, w_r)
    elif stage == "forward": f.forward(x, w1, w2)
    else: f.backward(x, w1, w2, w_r, dy, want_dgate=True)
    torch.cuda.synchronize()
    print(f"{stage}: {time.time()-t:.3f}s", flush=True)
got = {n: getattr(f.route_buf, n).cpu().numpy() for n in ("logits", "topk_idx")}
got.update(y=f.y.float().cpu().numpy(), dx=f.dx.float().cpu().numpy(), dw1=f.dw1.cpu().numpy(),
           dw2=f.dw2.cpu().numpy(), dw_r=f.dw_r.cpu().numpy(), dgate=f.dgate.cpu().numpy())
if skip_oracle: sys.exit(0)
import oracle
t = time.time()
lg = oracle.router(inp["x"], inp["w_r"])
ref = oracle_run(oracle, cfg, inp, lg, got["topk_idx"])
print(f"oracle: {time.time()-t:.1f}s threads={oracle.max_threads()}", flush=True)
for n in ("y", "dx", "dw1", "dw2", "dw_r", "dgate"):
    print(n, relerr(got[n], ref[n]))

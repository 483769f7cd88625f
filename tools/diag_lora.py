"""LoRA parity diagnostics: errors per output for a few shapes (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synthetic as S
import oracle as orc
from test_gpu_lora import gpu_run_lora, oracle_lora
from helpers import relerr

cases = [("opt", S.CONFIGS["opt"], 400), ("opt_gelu", S.CONFIGS["opt"].with_(act=S.ACT_GELU), 400),
         ("bert_relu", S.CONFIGS["bert"].with_(act=S.ACT_RELU), 400), ("bert", S.CONFIGS["bert"], 400),
         ("opt_T2000", S.CONFIGS["opt"], 2000), ("llama", S.CONFIGS["llama"], 300)]
for name, cfg, T in cases:
    inp = S.make_inputs(cfg, T)
    lora = S.make_lora(cfg, 16)
    got = gpu_run_lora(cfg, T, inp, lora, 16)
    lg = orc.router(inp["x"], inp["w_r"])
    ref = oracle_lora(orc, cfg, inp, lora, lg, got["topk_idx"])
    errs = {n: relerr(got[n].reshape(np.shape(ref[n])), ref[n]) for n in ("y", "dx", "dgate", "dw_r", "db1", "dc1", "db2", "dc2")}
    print(name, T, " ".join(f"{n}={e:.2e}" for n, e in errs.items()), flush=True)
    if errs["dc1"] > 0.02:
        g = got["dc1"].reshape(np.shape(ref["dc1"])); r = ref["dc1"]
        bad = np.argwhere(np.abs(g - r) > 0.05 * np.abs(r).max())
        print("  bad dc1 entries", len(bad), "of", r.size, bad[:10].tolist())
        D, bw = cfg.D, cfg.bw
        rows = np.unique(bad[:, -2]) if len(bad) else []
        print("  blocks", np.unique(np.asarray(rows) // bw)[:20])

"""Small LoRA and top-L invocations for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import synthetic as S
import paper_2312_10365_b200 as P
from test_gpu_lora import gpu_run_lora

what = sys.argv[1]
if what == "lora":
    for cfg, T in ((S.CONFIGS["bert"], 300), (S.FfnConfig("g8k4", 512, 4096, 8, 4, 200, "bf16", S.ACT_RELU), 200),
                   (S.CONFIGS["llama"].with_(G=86), 130)):
        gpu_run_lora(cfg, T, S.make_inputs(cfg, T), S.make_lora(cfg, 16), 16)
else:
    for causal, M, E in ((False, 8, 16), (True, 16, 16), (True, 13, 200)):
        tc = S.TOPL_CONFIGS["topl_tiny"].with_(n=300, M=M, E=E, causal=causal)
        cq, ck = S.make_pq_codes(tc)
        P.spt_mha_topl(torch.from_numpy(cq).cuda(), torch.from_numpy(ck).cuda(), 37, causal,
                       n_codewords=E)
torch.cuda.synchronize()
print("ok", what)

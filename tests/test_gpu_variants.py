"""GPU parity of the library's alternative kernel paths (selected by environment
knobs read once per process, so each case runs in its own interpreter):
  SPT_FFN_DAT=0       a7 with tokens on M (N = bw), fused epilogue (CTA-pair gather kernel)
  SPT_FFN_DAT=1       a7 with tokens on N + da_post_kernel
  SPT_FFN_DAT=2       a7 with tokens on N, per-(row, unit) fused epilogue
  (default SPT_FFN_DAT=3: tokens on N, row-major fused epilogue)
  SPT_FFN_G1_ROWS=128|32  1-CTA gathered kinds: TMA / cp.async row split of a 256-row stage
  SPT_FFN_PAIR_CPW=4  pair gather kernel with 4 cp.async / 8 epilogue warps (default 8 / 4)
  SPT_FFN_BWD_STREAMS=1|0  weight-gradient branch of the backward on a side stream always / never
                      (default: when dW1 has <= 4 tiles per SM, i.e. bert / tiny here)
  SPT_FFN_PREFETCH=1  L2 prefetch of gathered rows
  SPT_FFN_PAIR=1|0    CTA-pair (cta_group::2) weight-resident kernel for FWD2 + dX / neither (default: dX only)
  SPT_FFN_PAIR_GATHER=0  1-CTA FWD1 / dA kernel (default: CTA-pair gather kernel)
  SPT_FFN_SIMT=1      fp32 on the SIMT (FFMA) kernels instead of the split tensor-core path
  SPT_FFN_PDL=1       programmatic dependent launch of the hot-path kernels
  SPT_FFN_MLP=1       fused FWD1 -> FWD2 CTA-pair kernel (SwiGLU, bw = 128)
  SPT_FFN_DW_NG=3|5   dW raster groups of 3 / 5 N tiles (d = 4096: a ragged last group)
  SPT_FFN_PAIR_ROWS=0|128|20  pair FWD1 / dA stages gathered all by cp.async / all by TMA / a 5-call TMA split
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import oracle, synthetic as S
from helpers import TOL, gpu_run, oracle_run, relerr
for name, T in (("bert", 700), ("llama", 300), ("tiny", 333)):
    cfg = S.CONFIGS[name]
    inp = S.make_inputs(cfg, T)
    got = gpu_run(cfg, T, inp)
    lg = oracle.router(inp["x"], inp["w_r"])
    ref = oracle_run(oracle, cfg, inp, lg, got["topk_idx"])
    errs = {{n: relerr(got[n], ref[n]) for n in ("y", "dx", "dw1", "dw2", "dw_r", "dgate")}}
    assert all(e <= TOL[cfg.dtype] for e in errs.values()), (name, errs)
print("ok")
"""


@pytest.mark.parametrize("env", [{"SPT_FFN_DAT": "0"}, {"SPT_FFN_DAT": "1"}, {"SPT_FFN_DAT": "2"},
                                 {"SPT_FFN_G1_ROWS": "128"}, {"SPT_FFN_G1_ROWS": "32"}, {"SPT_FFN_PREFETCH": "1"}, {"SPT_FFN_PAIR": "1"}, {"SPT_FFN_PAIR": "0"},
                                 {"SPT_FFN_PAIR_GATHER": "0"}, {"SPT_FFN_SIMT": "1"}, {"SPT_FFN_PDL": "1"}, {"SPT_FFN_MLP": "1"},
                                 {"SPT_FFN_DW_NG": "3"}, {"SPT_FFN_DW_NG": "5"},
                                 {"SPT_FFN_PAIR_ROWS": "0"}, {"SPT_FFN_PAIR_ROWS": "128"},
                                 {"SPT_FFN_PAIR_ROWS": "20"}, {"SPT_FFN_PAIR_CPW": "4"},
                                 {"SPT_FFN_PAIR_CPW": "4", "SPT_FFN_DAT": "0"},
                                 {"SPT_FFN_BWD_STREAMS": "1"}, {"SPT_FFN_BWD_STREAMS": "0"}])
def test_variant_parity(env):
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_fused_fwd1_fwd2_many_tiles():
    """SPT_FFN_MLP=1 at a T where every cluster runs several pair tiles (both TMEM
    buffers in turn, chunk drains of tile n-2 gating FWD1 of tile n) and buckets
    end in ragged tiles."""
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests")).replace(
        'for name, T in (("bert", 700), ("llama", 300), ("tiny", 333)):', 'for name, T in (("llama", 3001),):')
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "SPT_FFN_MLP": "1"},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("dat", ["0", "1", "2", "3"])
def test_dat_many_tiles(dat):
    """Tokens-on-N a7 at T where every CTA runs several pair tiles (both TMEM
    buffers, the cross-warp dgate exchange reused tile after tile), ragged bucket
    ends, bw = 96 (bert: unit quarter 3 idle) and bw = 128 SwiGLU (llama)."""
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests")).replace(
        'for name, T in (("bert", 700), ("llama", 300), ("tiny", 333)):',
        'for name, T in (("llama", 3001), ("bert", 5003), ("opt", 2222)):')
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "SPT_FFN_DAT": dat},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr

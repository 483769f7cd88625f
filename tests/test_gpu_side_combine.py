"""GPU: the a8 grad-input combine as side work of the dW kernels (SPT_FFN_SIDE=1,
opt-in: measured slower) against the stand-alone combine kernel
(the default, SPT_FFN_SIDE=0).

Both sum each token's k partial rows in ascending j and then add the router
term in ascending j (combine.cu, reading c12), so dx must be BIT-identical, and
so must every other output (the dW kernels' own arithmetic does not change).
Each setting runs in its own interpreter (the knob is read once per process).
The oracle check of the default path is the rest of the suite; here also the
side path against the oracle at one size where every CTA claims many units."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import synthetic as S
from helpers import gpu_run
cfg = S.CONFIGS[{name!r}]
if {gate_none}:
    import dataclasses
    cfg = dataclasses.replace(cfg, gate=S.GATE_NONE)
inp = S.make_inputs(cfg, {T})
got = gpu_run(cfg, {T}, inp)
np.savez({out!r}, **{{n: got[n] for n in ("y", "dx", "dw1", "dw2", "dw_r", "dgate", "topk_idx")}})
print("ok")
"""


def _run(tmp_path, name, T, side, gate_none=False):
    out = str(tmp_path / f"{name}_{T}_{side}_{int(gate_none)}.npz")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), name=name, T=T, out=out,
                         gate_none=gate_none)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "SPT_FFN_SIDE": side},
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
    return dict(np.load(out))


@pytest.mark.parametrize("name,T,gate_none", [("bert", 3001, False), ("opt", 2000, False),
                                              ("llama", 5000, False), ("llama", 777, True),
                                              ("bert", 1, False), ("bert", 0, False)])
def test_side_combine_bit_identical(tmp_path, name, T, gate_none):
    a = _run(tmp_path, name, T, "1", gate_none)
    b = _run(tmp_path, name, T, "0", gate_none)
    for n in ("topk_idx", "y", "dx", "dw1", "dw2", "dw_r", "dgate"):
        assert a[n].shape == b[n].shape, n
        assert np.array_equal(a[n].view(np.uint8), b[n].view(np.uint8)), n


def test_side_combine_oracle_many_units(tmp_path):
    """The side path's dx against the oracle: llama (k = 22, d = 4096: 16 units
    per token) at T = 4096, where every CTA of both dW kernels claims tokens and
    the drain finishes the rest; sampled tokens, the oracle on its own fp64
    router logits with the GPU's (verified elsewhere) selection."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import synthetic as S
    from helpers import TOL, oracle_run, relerr
    cfg = S.CONFIGS["llama"]
    T = 4096
    got = _run(tmp_path, "llama", T, "1")
    inp = S.make_inputs(cfg, T)
    lg = oracle.router(inp["x"], inp["w_r"])
    tokens = np.random.default_rng(5).choice(T, 96, replace=False)
    ref = oracle_run(oracle, cfg, inp, lg, got["topk_idx"], tokens=tokens, blocks=[0])
    assert relerr(got["dx"][tokens], ref["dx"][tokens]) <= TOL[cfg.dtype]

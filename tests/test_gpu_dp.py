"""The N > 1 data-parallel path executed on ONE GPU (the box has a
single B200, and NCCL refuses two ranks on one device): two ranks (processes)
share cuda:0 over the gloo backend and run bench.py's real step --

  RoutedFFN on the rank's dp.shard_range token shard, the weight gradients on
  dp.attach_flat_grads' flat buffer, dp.OverlappedAllReduce started on its own
  stream at the event spt_ffn_backward records once dW is final (overlapping
  the grad-input kernels), the next step's backward waiting for it, and
  dp.max_over_ranks on CUDA tensors --

then every rank's all-reduced dw1 | dw2 | dw_r must equal the oracle's
full-batch gradient (reading c16: SUM over ranks = full batch) and its y / dx
rows the oracle's rows of its shard, at the bf16 bound 2e-2 (reading c14).
The oracle runs on its own fp64 logits with the GPU's (verified) selection.
A second case runs bench.py itself as 2 torchrun ranks (--backend gloo) and
checks its JSON line.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synthetic as S
from helpers import TOL, relerr

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = S.CONFIGS["llama"]   # the bench's model family (SwiGLU, G = 86, k = 22)
T_GLOBAL = 700


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    import paper_2312_10365_b200 as P
    from paper_2312_10365_b200 import dp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inp = S.make_inputs(CFG, T_GLOBAL)
    t0, t1 = dp.shard_range(T_GLOBAL, rank, world)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()  # noqa: E731
    x, dy = dev(inp["x"][t0:t1]), dev(inp["dy"][t0:t1])
    w1, w2, w_r = dev(inp["w1"]), dev(inp["w2"]), dev(inp["w_r"])
    f = P.RoutedFFN(t1 - t0, CFG.d, CFG.D, CFG.G, CFG.k, torch.bfloat16, CFG.act, CFG.gate)
    fg = dp.attach_flat_grads(f)
    ar = dp.OverlappedAllReduce(fg)
    assert ar.active
    for _ in range(2):  # bench.py's step, twice: the 2nd backward waits for the 1st all-reduce
        f.route(x, w_r)
        f.forward(x, w1, w2)
        ar.wait()
        f.backward(x, w1, w2, w_r, dy, dw_event=ar.event, want_dgate=True)
        ar.launch()
    ar.wait()
    torch.cuda.synchronize()
    tmax = dp.max_over_ranks(float(rank + 1), device="cuda")
    out_q.put((rank, (t0, t1), tmax, {
        "y": f.y.float().cpu().numpy(), "dx": f.dx.float().cpu().numpy(),
        "topk_idx": f.route_buf.topk_idx.cpu().numpy(), "logits": f.route_buf.logits.cpu().numpy(),
        "dw1": fg["dw1"].cpu().numpy(), "dw2": fg["dw2"].cpu().numpy(), "dw_r": fg["dw_r"].cpu().numpy()}))
    dist.destroy_process_group()


def test_two_ranks_one_gpu_allreduce_equals_full_batch(orc):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    inp = S.make_inputs(CFG, T_GLOBAL)
    # routing per shard: bit-exact against the oracle on the shard's logits; the
    # full-batch selection is the shards' selections stacked (routing is per token)
    ti = np.concatenate([r[3]["topk_idx"] for r in res])
    gl = np.concatenate([r[3]["logits"] for r in res])
    assert np.array_equal(ti, orc.topk(gl, CFG.k))
    lg = orc.router(inp["x"], inp["w_r"])
    assert relerr(gl, lg) <= 1e-4
    full = orc.backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, inp["dy"], CFG.act, CFG.gate)
    y = orc.forward(inp["x"], inp["w1"], inp["w2"], lg, ti, CFG.act, CFG.gate)
    tol = TOL["bf16"]
    assert res[0][1][0] == 0 and res[0][1][1] == res[1][1][0] and res[1][1][1] == T_GLOBAL
    for rank, (t0, t1), tmax, got in res:
        assert tmax == 2.0
        for n in ("dw1", "dw2", "dw_r"):
            assert relerr(got[n], full[n]) <= tol, (rank, n)
        assert relerr(got["y"], y[t0:t1]) <= tol
        assert relerr(got["dx"], full["dx"][t0:t1]) <= tol
    # both ranks hold the identical reduced buffer
    for n in ("dw1", "dw2", "dw_r"):
        assert np.array_equal(res[0][3][n], res[1][3][n])


def test_bench_two_ranks_gloo():
    """bench.py under torchrun with 2 ranks on one GPU (gloo): the N > 1 code of
    the bench (init, shard offsets, overlapped all-reduce, barrier + max over
    ranks) runs; strong scaling splits the config's tokens over the ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--config", "bert", "--scaling", "strong",
           "--steps", "3", "--warmup", "3", "--no-e2e", "--no-profile"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong" and rec["config"]["global_tokens"] == 8192
    assert rec["config"]["tokens_per_gpu"] == 4096 and rec["value"] > 0 and rec["gpu_launches"] > 0

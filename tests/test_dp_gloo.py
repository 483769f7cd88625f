"""Data-parallel host logic on CPU with gloo, world_size 2.

Token-sharded DP: each rank owns a contiguous token shard, computes its
shard's weight gradients, and one SUM all-reduce of the flat fp32 gradient
buffer (paper_2312_10365_b200.dp) must give the full-batch gradient (reading
c16), while per-token outputs are independent of the world size.  The per-rank
compute here is the CPU oracle (test infrastructure), so the test exercises
exactly the sharding / flat-buffer / all-reduce / max-over-ranks code that
bench.py runs over NCCL on the GPU box.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic as S
from paper_2312_10365_b200 import dp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_SWIGLU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    t0, t1 = dp.shard_range(T, rank, world)
    sh = {n: inp[n][t0:t1] for n in ("x", "dy")}
    lg = oracle.router(sh["x"], inp["w_r"])
    ti = oracle.topk(lg.astype(np.float32), cfg.k)
    g = oracle.backward(sh["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, sh["dy"], cfg.act, cfg.gate)
    fg = dp.FlatGrads({"dw1": g["dw1"].shape, "dw2": g["dw2"].shape, "dw_r": g["dw_r"].shape}, device="cpu")
    for n in ("dw1", "dw2", "dw_r"):
        fg[n].copy_(torch.from_numpy(g[n].astype(np.float32)))
    dp.allreduce_grads(fg)
    tmax = dp.max_over_ranks(float(rank + 1))
    out_q.put((rank, {n: fg[n].numpy().copy() for n in ("dw1", "dw2", "dw_r")}, g["dx"], (t0, t1), tmax))
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [64, 67])
def test_allreduce_equals_full_batch(orc, T):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_SWIGLU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    lg = orc.router(inp["x"], inp["w_r"])
    ti = orc.topk(lg.astype(np.float32), cfg.k)
    full = orc.backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, inp["dy"], cfg.act, cfg.gate)
    for rank, grads, dx, (t0, t1), tmax in res:
        assert tmax == 2.0                                     # max over ranks
        for n in ("dw1", "dw2", "dw_r"):                       # SUM over ranks == full batch
            np.testing.assert_allclose(grads[n], full[n], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(dx, full["dx"][t0:t1], rtol=1e-12, atol=1e-12)  # per-token independence
    # shards tile [0, T) exactly
    assert res[0][3][0] == 0 and res[0][3][1] == res[1][3][0] and res[1][3][1] == T


def test_shard_range_properties():
    for T in (0, 1, 7, 4096, 32768):
        for world in (1, 2, 3, 8):
            r = [dp.shard_range(T, i, world) for i in range(world)]
            assert r[0][0] == 0 and r[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def test_flat_grads_views_share_storage():
    fg = dp.FlatGrads({"dw1": (2, 3, 4), "dw2": (3, 4), "dw_r": (2, 4)}, device="cpu")
    fg.flat.zero_()
    fg["dw2"].fill_(1.0)
    assert fg.flat.sum().item() == 12.0
    assert fg["dw1"].data_ptr() == fg.flat.data_ptr()
    assert dp.allreduce_grads(fg) is None        # single process: no-op


class _FakeLoRA:
    """The gradient attributes of a RoutedLoRAFFN (dp.attach_flat_grads's LoRA branch)."""

    def __init__(self, shapes, G, d):
        self.grads = {n: torch.empty(s) for n, s in shapes.items()}
        self.dw_r = torch.empty(G, d)


def _lora_worker(rank, world, port, T, out_q):
    import oracle
    from oracle import lora as OL
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_SWIGLU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    lo = S.make_lora(cfg, 4)
    t0, t1 = dp.shard_range(T, rank, world)
    x, dy = inp["x"][t0:t1], inp["dy"][t0:t1]
    lg = oracle.router(x, inp["w_r"])
    ti = oracle.topk(lg.astype(np.float32), cfg.k)
    g = OL.lora_backward(x, inp["w1"], inp["w2"], inp["w_r"], lo, lg, ti, dy, cfg.act, cfg.gate)
    f = _FakeLoRA({n: g[n].shape for n in ("db1", "dc1", "db2", "dc2")}, cfg.G, cfg.d)
    fg = dp.attach_flat_grads(f, device="cpu")
    for n in ("db1", "dc1", "db2", "dc2"):
        f.grads[n].copy_(torch.from_numpy(g[n].astype(np.float32)))
    f.dw_r.copy_(torch.from_numpy(g["dw_r"].astype(np.float32)))
    assert f.grads["db1"].data_ptr() == fg.flat.data_ptr()  # views of the one flat buffer
    dp.allreduce_grads(fg)
    out_q.put((rank, {n: f.grads[n].numpy().copy() for n in f.grads} | {"dw_r": f.dw_r.numpy().copy()}))
    dist.destroy_process_group()


def test_lora_allreduce_equals_full_batch(orc):
    """LoRA-wrapped FFN: the flat buffer carries the factor gradients and
    dW_R (W is frozen); SUM over token shards = the full-batch gradients."""
    import oracle
    from oracle import lora as OL
    world, T = 2, 50
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lora_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_SWIGLU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    lo = S.make_lora(cfg, 4)
    lg = oracle.router(inp["x"], inp["w_r"])
    ti = oracle.topk(lg.astype(np.float32), cfg.k)
    full = OL.lora_backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lo, lg, ti, inp["dy"], cfg.act,
                            cfg.gate)
    for n in ("db1", "dc1", "db2", "dc2", "dw_r"):
        ref = np.asarray(full[n], np.float64)
        for r in range(world):
            got = res[r][n].astype(np.float64).reshape(ref.shape)
            assert np.max(np.abs(got - ref)) <= 1e-5 * max(1.0, np.max(np.abs(ref))), n


def _balance_worker(rank, world, port, T, lam, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_GELU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    t0, t1 = dp.shard_range(T, rank, world)
    x, dy = inp["x"][t0:t1], inp["dy"][t0:t1]
    lg = oracle.router(x, inp["w_r"])
    ti = oracle.topk(lg.astype(np.float32), cfg.k)
    g = oracle.backward(x, inp["w1"], inp["w2"], inp["w_r"], lg, ti, dy, cfg.act, cfg.gate, lb_weight=lam)
    fg = dp.FlatGrads({"dw1": g["dw1"].shape, "dw2": g["dw2"].shape, "dw_r": g["dw_r"].shape}, device="cpu")
    for n in ("dw1", "dw2", "dw_r"):
        fg[n].copy_(torch.from_numpy(g[n].astype(np.float32)))
    dp.allreduce_grads(fg)
    out_q.put((rank, fg["dw_r"].numpy().copy()))
    dist.destroy_process_group()


def test_balance_loss_is_per_shard(orc):
    """dp.py's documented semantics of the load-balancing term under DP: the SUM
    all-reduce gives sum_r lambda dL_r/dW_R with L_r the shard's own loss (its
    f_g, pbar_g) -- equal to the sum of per-shard oracle gradients and NOT the
    gradient of the global batch's loss."""
    world, T, lam = 2, 80, 0.5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_balance_worker, args=(r, world, port, T, lam, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = S.CONFIGS["tiny"].with_(act=S.ACT_GELU, d=64, D=256, G=8, k=3)
    inp = S.make_inputs(cfg, T)
    per_shard = 0
    for r in range(world):
        t0, t1 = dp.shard_range(T, r, world)
        lg = orc.router(inp["x"][t0:t1], inp["w_r"])
        ti = orc.topk(lg.astype(np.float32), cfg.k)
        per_shard = per_shard + orc.backward(inp["x"][t0:t1], inp["w1"], inp["w2"], inp["w_r"], lg, ti,
                                             inp["dy"][t0:t1], cfg.act, cfg.gate, lb_weight=lam)["dw_r"]
    lg = orc.router(inp["x"], inp["w_r"])
    ti = orc.topk(lg.astype(np.float32), cfg.k)
    glob = orc.backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, inp["dy"], cfg.act, cfg.gate,
                        lb_weight=lam)["dw_r"]
    for r in range(world):
        np.testing.assert_allclose(res[r], per_shard, rtol=1e-5, atol=1e-6)
    assert np.max(np.abs(per_shard - glob)) > 1e-4 * np.max(np.abs(glob))  # the readings differ

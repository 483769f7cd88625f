#!/usr/bin/env python
"""Benchmark of the SPT routed FFN (arXiv 2312.10365) on B200.

One "step" = the whole hot path of SURVEY §8(a) over one batch of synthetic
tokens resident in HBM: route (router GEMM, top-k, bucketing) -> forward
(gather-fused grouped GEMMs + combine) -> backward (dA/dZ, dX, dW1, dW2, dW_R)
-> (N > 1) one NCCL SUM all-reduce of the flat fp32 weight gradients.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama_scale]
  python bench.py --impl reference ...     (the CPU oracle as the reference arm)

Default workload: BASELINE.json configs[4] "LLaMA-7B FFN token-sharded scaling
run ... seq 4096" -- d=4096, D=11008 (SwiGLU), G=86, k=22, 8 x 4096 tokens per
GPU (weak scaling), bf16 storage / fp32 accumulate, random-init weights and
random tokens ("Random" workload).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthetic as S  # noqa: E402

METRIC = "routed-FFN fwd+bwd tokens/s at 1/2/4/8 B200; tensor-pipe % of bf16 peak"
UNIT = "tokens/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"],
                "bf16_sustained": d["bf16_tflops_sustained"], "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0,
            "src": "fallback (B200_PROFILING.md)"}


# --------------------------------------------------------------- work model
def kernel_work(cfg, T):
    """Algorithmic FLOPs (tensor kernels) or bytes (HBM kernels) per launch,
    per SURVEY §8(d): GEMM work counts only activated blocks."""
    P = T * cfg.k
    mp, bw, d, G = cfg.mprime, cfg.bw, cfg.d, cfg.G
    e = 2 if cfg.dtype == "bf16" else 4
    return {
        "tc_router": ("tensor", 2.0 * T * d * G),
        "tc_fwd1_gate_up": ("tensor", 2.0 * P * mp * bw * d),
        "tc_fwd2_down": ("tensor", 2.0 * P * bw * d),
        "tc_bwd_dA": ("tensor", 2.0 * P * bw * d),
        "tc_bwd_dAT": ("tensor", 2.0 * P * bw * d),  # a7, tokens on N (default for bw <= 128)
        "tc_bwd_dX": ("tensor", 2.0 * P * mp * bw * d),
        "tc_bwd_dW1": ("tensor", 2.0 * P * mp * bw * d),
        "tc_bwd_dW2": ("tensor", 2.0 * P * bw * d),
        "tc_bwd_dWR": ("tensor", 2.0 * P * d),
        "combine_fwd": ("hbm", P * d * e + 8.0 * P + T * d * e),
        "combine_bwd": ("hbm", P * d * e + 12.0 * P + T * d * e),
        "topk_hist": ("hbm", 4.0 * T * G + 8.0 * T * cfg.k),
        "bucket_scatter": ("hbm", 20.0 * P),
        # fp32 on tensor cores (reading c13'): fp32 -> bf16 hi | lo copies of x (route,
        # forward, backward), dy, w1, w2 (forward, backward) and w_r (route); 4 bytes read
        # + 4 written per element, averaged over the step's 9 launches
        "split_bf16": ("hbm", 8.0 * (3 * T * d + T * d + 2 * (mp * cfg.D * d + cfg.D * d) + G * d) / 9),
        # fp32 path (tiny config): CUDA-core FFMA kernels, no tensor cores (reading c13)
        "simt_f1": ("alu", 2.0 * P * mp * bw * d),
        "simt_f2": ("alu", 2.0 * P * bw * d),
        "simt_b1": ("alu", 2.0 * P * bw * d),
        "simt_dw": ("alu", (2.0 * P * mp * bw * d + 2.0 * P * bw * d) / 2),  # dW1, dW2: mean per launch
        "simt_b2": ("alu", 2.0 * P * mp * bw * d),
    }


FP32_FMA_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # TFLOP/s: 128 FP32 lanes/SM x 2 FLOP x SMs x max clock


def step_gemm_flops(cfg, T, lora=0):
    """fwd 2(m'+1) d bw k + bwd 2x that, per token, + router 6 d G.
    LoRA rank r: W frozen, so the bwd is dA + dX only (1x fwd), plus the
    rank-r terms: per pair 2 bw r (2 m' + 1) fwd and 2 bw r (2 m' + 2) bwd, per
    token 2 d r (m' + 1) fwd and 2 d r (2 m' + 2) bwd."""
    mp, d, bw, k = cfg.mprime, cfg.d, cfg.bw, cfg.k
    fwd = 2.0 * (mp + 1) * d * bw * k
    if not lora:
        return (fwd * 3 + 6.0 * d * cfg.G) * T
    r = lora
    extra = k * 2.0 * bw * r * (4 * mp + 3) + 2.0 * d * r * (3 * mp + 3)
    return (fwd * 2 + 6.0 * d * cfg.G + extra) * T


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception as ex:  # nvidia-smi missing: report no clocks
            log("clock sampler unavailable:", ex)
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), p[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i in range(4) if r[i].lower() == "active"})
        sm = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows),
                "sm_mhz_min": min(sm), "samples": len(rows), "reasons": reasons}


# ----------------------------------------------------------------- oracle
def oracle_sample(cfg, n_tok, lora=0):
    """The CPU oracle (as it stands) over route + fwd + bwd of `n_tok` tokens of
    the workload (LoRA rank > 0: oracle/lora.py's fwd + bwd); returns (seconds, threads)."""
    import oracle
    inp = S.make_inputs(cfg, n_tok)
    lo = S.make_lora(cfg, lora) if lora else None
    t = time.perf_counter()
    lg = oracle.router(inp["x"], inp["w_r"])
    ti = oracle.topk(lg.astype(np.float32), cfg.k)
    oracle.bucket(ti, cfg.G)
    if lora:
        from oracle import lora as OL
        OL.lora_forward(inp["x"], inp["w1"], inp["w2"], lo, lg, ti, cfg.act, cfg.gate)
        OL.lora_backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lo, lg, ti, inp["dy"], cfg.act,
                         cfg.gate)
    else:
        oracle.forward(inp["x"], inp["w1"], inp["w2"], lg, ti, cfg.act, cfg.gate)
        oracle.backward(inp["x"], inp["w1"], inp["w2"], inp["w_r"], lg, ti, inp["dy"], cfg.act,
                        cfg.gate)
    return time.perf_counter() - t, oracle.max_threads()


def cpu_baseline(cfg, target_s=15.0, lora=0):
    """Oracle on a token sample sized (two calibration rounds) to ~target_s."""
    n, (secs, cores) = 16, oracle_sample(cfg, 16, lora)
    for _ in range(2):
        if secs >= 0.6 * target_s or n >= 8192:
            break
        n = int(max(16, min(8192, n * target_s / max(secs, 1e-3))))
        secs, cores = oracle_sample(cfg, n, lora)
    what = (f"LoRA rank {lora}: fp64 numpy oracle (oracle/lora.py, BLAS threads)" if lora else
            f"all {cfg.G} blocks' dW), {secs:.1f} s, fp64 C oracle, OpenMP")
    return {"value": n / secs, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} tokens of {cfg.name} (route+fwd+bwd, " + what
            + (f", {secs:.1f} s" if lora else "")}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # calibrate the sample like cpu_baseline (a probe large enough that the oracle's
    # per-call fixed costs do not dominate), then fit steps + warmup into ~150 s
    budget = 150.0 / max(1, args.steps + args.warmup)          # seconds per step
    n0 = 64
    t0, _ = oracle_sample(cfg, n0, args.lora)
    n = int(max(8, min(2048, n0 * budget / max(t0, 1e-3))))
    for _ in range(args.warmup):
        oracle_sample(cfg, n, args.lora)
    tot, cores = 0.0, 1
    for _ in range(args.steps):
        s, cores = oracle_sample(cfg, n, args.lora)
        tot += s
    value = n * args.steps / tot
    sample = f"{n} tokens of {cfg.name} per step (route+fwd+bwd, fp64 C oracle, OpenMP)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg, args.gpus, cfg.T, args.balance_weight, args.lora),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------ f4: top-L selection (Alg. 3)
TOPL_METRIC = "sparse-MHA top-L selection (Alg. 3) queries/s"


def topl_eq3_ops(cfg):
    """Algorithmic work of Eq. 3 over one selection, independent of
    how the kernel packs codes: per (query, candidate key) pair, M code equality
    tests and M - 1 additions of their indicators (2M - 1 integer ops); candidates =
    n (bidirectional) or q + 1 (causal).  The bucket sort of Alg. 3 adds O(L) per
    query on top (not counted)."""
    pairs = cfg.n * (cfg.n + 1) / 2 if cfg.causal else float(cfg.n) * cfg.n
    return cfg.heads * pairs * (2.0 * cfg.M - 1)


def topl_alu_ops(cfg):
    """The kernel's own instruction recipe (implementation ops, not algorithmic):
    per (query, candidate key) pair 6 ALU ops per packed code word (XOR, AND, ADD,
    OR, AND, POPC -- the zero-field test) plus 1 ADD; words = ceil(M / 8) for E <= 16
    (nibbles), else ceil(M / 4) (bytes); candidates = n (bidirectional) or q+1 (causal)."""
    pairs = cfg.n * (cfg.n + 1) / 2 if cfg.causal else float(cfg.n) * cfg.n
    cpw = 8 if cfg.E <= 16 else 4
    return cfg.heads * pairs * 7.0 * ((cfg.M + cpw - 1) // cpw)


def topl_workload(cfg, world):
    return {"workload": f"{cfg.name}: top-L over PQ codes, {cfg.heads} (sequence, head) problems x "
                        f"n={cfg.n} queries/keys, M={cfg.M} codebooks, E={cfg.E}, L={cfg.L} "
                        f"(lambda={cfg.lam}), {'causal' if cfg.causal else 'bidirectional'}",
            "queries_per_gpu": cfg.heads * cfg.n, "parallelism": f"dp{world}",
            "l2": "L2 flushed (256 MB write) before every timed launch; codes %.0f MB, indices %.0f MB" % (
                2 * cfg.heads * cfg.n * cfg.M / 1e6, cfg.heads * cfg.n * cfg.L * 4 / 1e6)}


def topl_oracle_sample(cfg, n_heads, n_q):
    from oracle import topl as OT
    cq, ck = S.make_pq_codes(cfg, heads=n_heads)
    if cfg.causal:
        ck = cq
    t = time.perf_counter()
    for h in range(n_heads):
        OT.topl_by_sort(cq[h][:n_q], ck[h], cfg.L, cfg.causal)
    return time.perf_counter() - t


def run_topl(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank != 0:
            return
        nq = 64
        for _ in range(args.warmup):
            topl_oracle_sample(cfg, 1, nq)
        tot = sum(topl_oracle_sample(cfg, 1, nq) for _ in range(args.steps))
        value = nq * args.steps / tot
        sample = f"{nq} queries of one head per step (numpy closed-form oracle, 1 thread)"
        print(json.dumps({
            "impl": "reference", "metric": TOPL_METRIC, "value": value, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": topl_workload(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    import torch
    import torch.distributed as dist
    import paper_2312_10365_b200 as P
    from paper_2312_10365_b200 import dp
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cq, ck = S.make_pq_codes(cfg.with_(cfg_index=cfg.cfg_index + 100 * rank))  # per-rank sequences
    if cfg.causal:
        ck = cq
    a, b = torch.from_numpy(cq).cuda(), torch.from_numpy(ck).cuda()
    out = torch.empty(cfg.heads, cfg.n, cfg.L, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        P.spt_mha_topl(a, b, cfg.L, cfg.causal, out=out, n_codewords=cfg.E)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    if world > 1:
        dist.barrier()
    n0 = P.launch_count()
    evs = []
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush, outside the timed pair
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.spt_mha_topl(a, b, cfg.L, cfg.causal, out=out, n_codewords=cfg.E)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    launches = P.launch_count() - n0
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    clocks = sampler.stop()
    ms_max = dp.max_over_ranks(ms, device="cuda")
    q = cfg.heads * cfg.n
    # end to end: codes from pinned host, indices back to pinned host, every step
    ah, bh = a.cpu().pin_memory(), b.cpu().pin_memory()
    oh = torch.empty(out.shape, dtype=torch.int32).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        a.copy_(ah, non_blocking=True)
        b.copy_(bh, non_blocking=True)
        P.spt_mha_topl(a, b, cfg.L, cfg.causal, out=out, n_codewords=cfg.E)
        oh.copy_(out, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e = dp.max_over_ranks(e0.elapsed_time(e1) / args.steps, device="cuda")
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    f_hz = 1.965e9
    peak = 148 * 64 * f_hz / 1e9  # alu-pipe lanes/clk/SM x SMs x max clock, Gops/s
    ach = topl_eq3_ops(cfg) / (ms / 1e3) / 1e9
    res = {
        "metric": TOPL_METRIC, "value": q * world / (ms_max / 1e3), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded clustered PQ codes)",
        "config": topl_workload(cfg, world),
        "roofline": {"bound": "alu", "kernel": "topl_select", "achieved": ach, "peak": peak, "unit": "Gops/s",
                     "frac": ach / peak, "traffic": None,
                     "peak_src": "DESIGN.md: 64 alu-pipe lanes/clk/SM (B300_MICROARCH rt_SMSP=2) x 148 SMs "
                                 "x 1.965 GHz",
                     "algorithmic": "Eq. 3: 2M - 1 integer ops per (query, candidate key) pair",
                     "algorithmic_per_launch": topl_eq3_ops(cfg),
                     "implementation_ops_per_launch": topl_alu_ops(cfg),
                     "implementation_frac": topl_alu_ops(cfg) / (ms / 1e3) / 1e9 / peak},
        "gpu_launches": launches, "clocks": clocks,
        "e2e": {"value": q * world / (ms_e / 1e3), "unit": "queries/s", "ms_per_step": ms_e,
                "h2d_bytes_per_step": int(a.numel() + b.numel()), "d2h_bytes_per_step": int(out.numel() * 4)},
    }
    if world == 1 and not args.no_cpu_baseline:
        n_q = 256
        secs = topl_oracle_sample(cfg, 1, n_q)
        res["cpu_baseline"] = {"value": n_q / secs, "unit": "queries/s", "cores": 1, "kind": "oracle",
                               "sample": f"{n_q} queries of one head, numpy closed-form oracle, {secs:.1f} s"}
    print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def workload_config(cfg, world, T, balance_weight=0.0, lora=0):
    lb = f", load-balancing loss lambda={balance_weight}" if balance_weight else ""
    if lora:
        lb += f", LoRA rank {lora} on fc1/fc2 (W frozen: no dW1/dW2; factor grads)"
    return {"workload": f"{cfg.name}: routed FFN d={cfg.d} D={cfg.D} G={cfg.G} k={cfg.k} bw={cfg.bw} "
                        f"act={['relu', 'gelu', 'swiglu'][cfg.act]} "
                        f"gate={['sigmoid', 'none'][cfg.gate]}, {T} tokens per GPU{lb}",
            "tokens_per_gpu": T, "global_tokens": T * world, "parallelism": f"dp{world}",
            "l2": (("inputs larger than L2 (x, dy %.0f MB each; weights %.0f MB)" if not l2_flush(cfg, T)
                    else "L2 flushed (256 MB write, outside the timed events) before every timed step; "
                         "x, dy %.0f MB each, weights %.0f MB") % (
                T * cfg.d * (2 if cfg.dtype == 'bf16' else 4) / 1e6,
                (cfg.mprime + 1) * cfg.D * cfg.d * (2 if cfg.dtype == 'bf16' else 4) / 1e6))}


L2_BYTES = 126e6  # B200 L2 (B200_PROFILING.md)


def l2_flush(cfg, T):
    """Timing rule: inputs larger than L2, else flush L2 between timed steps.  x, dy
    and the weights together below 2x L2 -> flush."""
    e = 2 if cfg.dtype == "bf16" else 4
    return (2 * T * cfg.d + (cfg.mprime + 1) * cfg.D * cfg.d + cfg.G * cfg.d) * e < 2 * L2_BYTES


# ------------------------------------------------- other configs (summary)
def config_summary(names, steps=10, warmup=3):
    """Device-timed step of each named config (route + fwd + bwd through the C ABI,
    CUDA-graph replay, L2 flushed before every timed step when the inputs fit in L2):
    {name: {ms_per_step, tokens_per_s, tokens, dtype, l2_flushed}}."""
    import torch
    import paper_2312_10365_b200 as P
    res = {}
    fbuf = torch.empty(int(2 * L2_BYTES) // 4, dtype=torch.float32, device="cuda")
    for name in names:
        cfg = S.ALL_CONFIGS[name]
        try:
            T = cfg.T
            dt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
            inp = S.make_inputs(cfg, T)
            x, w1, w2, w_r, dy = (torch.from_numpy(inp[n]).to(dt).cuda()
                                  for n in ("x", "w1", "w2", "w_r", "dy"))
            del inp
            f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, dt, cfg.act, cfg.gate)

            def step():
                f.route(x, w_r)
                f.forward(x, w1, w2)
                f.backward(x, w1, w2, w_r, dy)
            for _ in range(warmup):
                step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            flush = l2_flush(cfg, T)
            tot = 0.0
            for _ in range(steps):
                if flush:
                    fbuf.fill_(1.0)
                e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_a.record()
                g.replay()
                e_b.record()
                torch.cuda.synchronize()
                tot += e_a.elapsed_time(e_b)
            ms = tot / steps
            res[name] = {"ms_per_step": ms, "tokens_per_s": T / (ms / 1e3), "tokens": T,
                         "dtype": cfg.dtype, "l2_flushed": flush,
                         "gemm_tflops": step_gemm_flops(cfg, T) / (ms / 1e3) / 1e12}
            del g, f, x, w1, w2, w_r, dy
            torch.cuda.empty_cache()
        except Exception as ex:  # a summary entry must not hide the headline
            res[name] = {"error": str(ex)[:200]}
    return res


# ------------------------------------------------------- dense context
def dense_lora_context(cfg, x, w1, w2, dy, lora, ms_routed, iters=5, warmup=2):
    """The dense LoRA FFN fwd+bwd at the same shape through cuBLAS (torch.matmul,
    W frozen: backward = dX + the LoRA factor gradients, no dW) -- the B200
    analogue of the paper's own comparison, LoRA vs SPT (Table 1's FFN time
    128.8 -> 54.9 ms, Table 5).  Context only: not this library's path."""
    import torch
    import torch.nn.functional as F
    D, mp = cfg.D, cfg.mprime
    w1 = w1.reshape(-1, cfg.d)                              # [m'D, d]
    b1 = lora["b1"].reshape(mp, -1, cfg.d)                  # [m', r, d]
    c1 = lora["c1"].reshape(mp, D, -1)                      # [m', D, r]
    b2, c2 = lora["b2"], lora["c2"]

    def act(z):
        if cfg.act == S.ACT_SWIGLU:
            return F.silu(z[:, :D]) * z[:, D:]
        return F.relu(z) if cfg.act == S.ACT_RELU else F.gelu(z)

    def step():
        xr = x.detach().requires_grad_(True)
        fac = [t.detach().requires_grad_(True) for t in (b1, c1, b2, c2)]
        B1, C1, B2, C2 = fac
        z = xr @ w1.t() + torch.cat([(xr @ B1[m].t()) @ C1[m].t() for m in range(mp)], dim=1)
        h = act(z)
        y = h @ w2 + (h @ B2) @ C2
        torch.autograd.grad(y, [xr] + fac, dy)

    for _ in range(warmup):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return {"ms_per_step": ms, "routed_speedup": ms / ms_routed, "ideal_speedup": cfg.G / cfg.k,
            "what": "dense LoRA FFN fwd+bwd (torch autograd on cuBLAS bf16; W frozen: dX + LoRA "
                    "factor grads), same T, d, D, rank"}


def dense_context(cfg, x, w1, w2, dy, ms_routed, iters=5, warmup=2):
    """the dense FFN fwd+bwd at the same shape through cuBLAS
    (torch.matmul, bf16 in / fp32 accumulate) + torch elementwise activation --
    the B200 analogue of the paper's dense-vs-SPT comparison (ideal speedup
    G/k).  Context only: not this library's path."""
    import torch
    import torch.nn.functional as F
    D = cfg.D
    w1 = w1.reshape(-1, cfg.d)  # [m'D, d] (SwiGLU: gate rows then up rows)

    def act(z):
        if cfg.act == S.ACT_SWIGLU:
            return F.silu(z[:, :D]) * z[:, D:]
        return F.relu(z) if cfg.act == S.ACT_RELU else F.gelu(z)

    def step():
        z = x @ w1.t()                      # [T, m'D]
        zr = z.detach().requires_grad_(True)
        h = act(zr)
        _ = h @ w2                          # Y [T, d]
        dh = dy @ w2.t()                    # [T, D]
        _ = h.t() @ dy                      # dW2 [D, d]
        (dz,) = torch.autograd.grad(h, zr, dh)
        _ = dz @ w1                         # dX [T, d]
        _ = dz.t() @ x                      # dW1 [m'D, d]

    for _ in range(warmup):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = 6.0 * x.shape[0] * cfg.d * D * (cfg.mprime + 1)
    return {"ms_per_step": ms, "gemm_tflops": flops / (ms / 1e3) / 1e12,
            "routed_speedup": ms / ms_routed, "ideal_speedup": cfg.G / cfg.k,
            "what": "dense FFN fwd+bwd (torch.matmul / cuBLAS bf16 + torch activation), same T, d, D"}


# ------------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama_scale", choices=sorted(S.ALL_CONFIGS))
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense cuBLAS context")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the summary of the other configs (default run only)")
    ap.add_argument("--balance-weight", type=float, default=0.0,
                    help="lambda of the load-balancing loss (SURVEY f2; 0 = the north_star step)")
    ap.add_argument("--topl", default="", choices=[""] + sorted(S.TOPL_CONFIGS),
                    help="time the sparse-MHA top-L selection (SURVEY f4, Alg. 3) on this "
                         "workload instead of the routed FFN")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="N=1 runs capture the step once into a CUDA graph and replay it (no "
                         "per-kernel launch gaps; the library's host-side argument checks and "
                         "tensor-map encodes run once, at capture); this flag times eager launches")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: lets several ranks share one GPU, "
                         "to exercise the multi-rank path where only one device is available)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the config's tokens on every rank; strong: the config's tokens split "
                         "over the ranks (dp.shard_range)")
    ap.add_argument("--lora", type=int, default=0, metavar="R",
                    help="LoRA-wrapped routed FFN of rank R (SURVEY f3; W frozen, factors trained); "
                         "0 = the north_star step")
    args = ap.parse_args()
    if args.topl:
        run_topl(args, S.TOPL_CONFIGS[args.topl])
        return
    cfg = S.ALL_CONFIGS[args.config]
    if args.tokens:
        cfg = cfg.with_(T=args.tokens)
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2312_10365_b200 as P
    from paper_2312_10365_b200 import dp

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())  # gloo: several ranks may share a device
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    if args.scaling == "strong":  # the config's global batch split over the ranks
        t0, t1 = dp.shard_range(cfg.T, rank, world)
        T, offset = t1 - t0, t0
        if offset % 1024:
            raise SystemExit("strong scaling needs shards that start at multiples of 1024 tokens")
    else:                         # the config's batch on every rank
        T = cfg.T
        offset = rank * ((T + 1023) // 1024) * 1024
    T_global = dp.shard_range(cfg.T, 0, 1)[1] if args.scaling == "strong" else T * world
    dt = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
    t_gen = time.time()
    inp = S.make_inputs(cfg, T, token_offset=offset)
    log(f"[rank {rank}] inputs generated in {time.time() - t_gen:.1f}s")
    dev = {n: torch.from_numpy(inp[n]).to(dt).cuda() for n in ("x", "w1", "w2", "w_r", "dy")}
    del inp
    x, w1, w2, w_r, dy = (dev[n] for n in ("x", "w1", "w2", "w_r", "dy"))
    lora = None
    if args.lora:
        lora = {n: torch.from_numpy(v).to(dt).cuda() for n, v in S.make_lora(cfg, args.lora).items()}
        f = P.RoutedLoRAFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, dt, cfg.act, args.lora, cfg.gate,
                            balance_weight=args.balance_weight)
    else:
        f = P.RoutedFFN(T, cfg.d, cfg.D, cfg.G, cfg.k, dt, cfg.act, cfg.gate,
                        balance_weight=args.balance_weight)
    fg = dp.attach_flat_grads(f)

    # N > 1: the dW all-reduce starts (side stream) at the event the backward
    # records once dw1/dw2/dw_r are final and overlaps its grad-input kernels;
    # the next step's backward waits for it before overwriting the gradients.
    ar = dp.OverlappedAllReduce(fg)

    def step():
        f.route(x, w_r)
        if args.balance_weight:
            f.balance_loss()  # the router's load-balancing loss of this routing
        if lora is None:
            f.forward(x, w1, w2)
            ar.wait()
            # single process: no event, so the library runs dX first and the
            # grad-input combine as side work of the dW kernels
            f.backward(x, w1, w2, w_r, dy, dw_event=ar.event if ar.active else None)
        else:
            f.forward(x, w1, w2, lora)
            ar.wait()
            f.backward(x, w1, w2, w_r, lora, dy, grad_event=ar.event)
        ar.launch()

    def barrier():
        if world > 1:
            dist.barrier()

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    ar.wait()
    torch.cuda.synchronize()
    run_step = step
    launches_per_step = None
    if args.graph and world == 1:
        try:
            n0 = P.launch_count()
            step()
            torch.cuda.synchronize()
            n1 = P.launch_count() - n0
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            graph.replay()
            torch.cuda.synchronize()
            run_step, launches_per_step = graph.replay, n1
        except Exception as ex:  # capture unsupported here: time eager launches
            log(f"[bench] CUDA graph capture failed ({ex}); timing eager launches")
            torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    flush = l2_flush(cfg, T)
    fbuf = torch.empty(int(2 * L2_BYTES) // 4, dtype=torch.float32, device="cuda") if flush else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush else 1)]
    barrier()
    torch.cuda.synchronize()
    n0 = P.launch_count()
    if flush:  # small inputs: every step from a flushed L2, each step timed on its own
        for e_a, e_b in evs:
            fbuf.fill_(1.0)
            e_a.record(stream)
            run_step()
            ar.wait()
            e_b.record(stream)
    else:      # inputs larger than L2: K steps back to back
        evs[0][0].record(stream)
        for _ in range(args.steps):
            run_step()
        ar.wait()
        evs[0][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = P.launch_count() - n0
    if launches_per_step is not None:  # graph replays bypass the host-side launch counter
        launches = launches_per_step * args.steps
    ms = sum(e_a.elapsed_time(e_b) for e_a, e_b in evs) / args.steps
    ms_max = dp.max_over_ranks(ms, device="cuda")
    value = T_global / (ms_max / 1e3)   # every rank's tokens / the slowest rank's time

    # ---- per-kernel device times (CUDA events around each library launch)
    prof = {}
    if not args.no_profile:
        P.profile_enable(True)
        for _ in range(args.steps):
            step()
        ar.wait()
        torch.cuda.synchronize()
        prof = P.profile_read()
        P.profile_enable(False)
    clocks = sampler.stop()

    # ---- end to end through the public API, host buffers: every step copies its
    # inputs x, dy from pinned host memory and its outputs y, dx back; the copies
    # of neighbouring steps overlap the kernels (paper_2312_10365_b200.pipeline)
    e2e = None
    if not args.no_e2e:
        from paper_2312_10365_b200.pipeline import HostStepPipeline
        xh = torch.empty_like(x, device="cpu").pin_memory()
        dyh = torch.empty_like(dy, device="cpu").pin_memory()
        xh.copy_(x)
        dyh.copy_(dy)
        yh = torch.empty_like(x, device="cpu").pin_memory()
        dxh = torch.empty_like(x, device="cpu").pin_memory()
        pipe = HostStepPipeline(f, w1, w2, w_r, grad_hook=lambda: dp.allreduce_grads(fg), lora=lora)
        pipe.step(0, xh, dyh, yh, dxh)
        pipe.synchronize()
        barrier()
        # steady-state period of the pipeline: from the end of warm-up step 2's D2H to the
        # end of the last timed step's D2H, i.e. exactly k2 steps, each with its own H2D,
        # kernels and D2H (the one-time fill / drain of the 3-stage pipeline is not a step)
        for i in range(1, 3):
            pipe.step(i, xh, dyh, yh, dxh)
        k2 = max(6, args.steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_d2h)
        for i in range(k2):
            pipe.step(3 + i, xh, dyh, yh, dxh)
        e1.record(pipe.s_d2h)
        pipe.synchronize()
        ms_e = dp.max_over_ranks(e0.elapsed_time(e1) / k2, device="cuda")
        # the same k2 steps from an idle pipeline: the first H2D and the last D2H
        # are not overlapped by anything (reported beside the steady-state value)
        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(pipe.s_h2d)
        for i in range(k2):
            pipe.step(3 + k2 + i, xh, dyh, yh, dxh)
        e3.record(pipe.s_d2h)
        pipe.synchronize()
        ms_fill = dp.max_over_ranks(e2.elapsed_time(e3) / k2, device="cuda")
        hb, db = pipe.bytes_per_step()
        e2e = {"value": T_global / (ms_e / 1e3), "unit": UNIT, "ms_per_step": ms_e,
               "ms_per_step_incl_fill_drain": ms_fill,
               "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db,
               "what": "per step: H2D x, dy from pinned host -> route/fwd/bwd(+allreduce) -> D2H y, dx "
                       "to pinned host; copies of adjacent steps overlap the kernels (copy streams); "
                       "steady-state period over k2 steps (pipeline fill / drain excluded); PCIe "
                       "ceiling on this box: 49.6 GB/s per direction with both directions busy "
                       "(tools/pcie_bw.py)", "steps": k2}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    pk = peaks()
    work = kernel_work(cfg, T)
    kernels = {}
    for name, (cnt, tot) in prof.items():
        per = tot / max(cnt, 1)
        kernels[name] = {"launches_per_step": cnt / args.steps, "ms_per_launch": per}
        if name in work:
            kind, amt = work[name]
            if kind in ("tensor", "alu"):
                kernels[name]["tflops"] = amt / (per / 1e3) / 1e12
            else:
                kernels[name]["gbs"] = amt / (per / 1e3) / 1e9
    roofline = None
    if prof:
        step_ms_prof = sum(t for _, t in prof.values()) / args.steps
        dom = max(prof, key=lambda n: prof[n][1])
        cnt, tot = prof[dom]
        per = tot / cnt
        kind, amt = work.get(dom, ("tensor", 0.0))
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r02c_ncu_traffic.json")
        # the capture is of the plain bf16 step: never attach it to a LoRA / other line
        if os.path.exists(tp) and cfg.name == "llama_scale" and T == 32768 and not args.lora \
                and not args.balance_weight:
            kt = json.load(open(tp))["kernels"].get(dom)
            if kt:
                traffic = kt["dram_read_bytes"] + kt["dram_write_bytes"]
        if kind == "alu":
            ach = amt / (per / 1e3) / 1e12
            roofline = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": FP32_FMA_PEAK,
                        "unit": "TFLOP/s", "frac": ach / FP32_FMA_PEAK, "traffic": traffic,
                        "peak_src": "fp32 FFMA: 148 SMs x 128 lanes x 2 FLOP x 1.965 GHz (B200 unit "
                                    "counts, max clock)",
                        "algorithmic_per_launch": amt, "ms_per_launch": per,
                        "share_of_step": tot / args.steps / step_ms_prof}
        elif kind == "tensor":
            ach = amt / (per / 1e3) / 1e12
            # fp32 (split path, reading c13'): every fp32 product is three bf16 tensor-core
            # products, so the fp32 roof is the measured bf16 rate / 3
            f32 = cfg.dtype == "f32"
            peak = pk["bf16_sustained"] / 3 if f32 else pk["bf16_sustained"]
            roofline = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": peak,
                        "unit": "TFLOP/s", "frac": ach / peak, "traffic": traffic,
                        "traffic_src": "profiles/r02c_ncu_traffic.json (dram read+write bytes per launch)",
                        "peak_src": pk["src"] + " bf16 sustained" +
                                    (" / 3 (fp32 as hi*hi + hi*lo + lo*hi bf16 products)" if f32 else ""),
                        "algorithmic_per_launch": amt, "ms_per_launch": per,
                        "share_of_step": tot / args.steps / step_ms_prof}
        else:
            ach = amt / (per / 1e3) / 1e9
            roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": ach / pk["hbm_gbs"], "traffic": traffic, "peak_src": pk["src"],
                        "algorithmic_per_launch": amt, "ms_per_launch": per,
                        "share_of_step": tot / args.steps / step_ms_prof}
    step_tf = step_gemm_flops(cfg, T, args.lora) / (ms_max / 1e3) / 1e12
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded random tokens and weights)",
        "config": dict(workload_config(cfg, world, T, args.balance_weight, args.lora),
                       **({"cuda_graph": True} if launches_per_step is not None else {}),
                       **({"backend": args.backend} if world > 1 else {}),
                       global_tokens=T_global),
        "tensor_pipe_frac_of_bf16_peak": {"step_gemm_tflops": step_tf, "peak": pk["bf16_sustained"],
                                          "frac": step_tf / pk["bf16_sustained"],
                                          "peak_src": pk["src"] + " bf16 sustained"},
        "roofline": roofline, "kernels": kernels, "gpu_launches": launches, "clocks": clocks, "e2e": e2e,
    }
    if world == 1 and not args.no_dense and cfg.dtype == "bf16":
        try:
            out["dense_context"] = (dense_lora_context(cfg, x, w1, w2, dy, lora, ms_max) if lora
                                    else dense_context(cfg, x, w1, w2, dy, ms_max))
        except Exception as ex:  # e.g. out of memory: context only
            out["dense_context"] = {"error": str(ex)[:200]}
    if world == 1 and args.config == "llama_scale" and not (args.tokens or args.lora or args.balance_weight
                                                               or args.no_configs):
        # the other BASELINE configs and the paper's own workloads, each timed the same
        # way (CUDA-graph step, L2 flushed between steps when the inputs fit in L2)
        del x, w1, w2, w_r, dy, f, fg, dev
        torch.cuda.empty_cache()
        out["other_configs"] = config_summary(
            ["tiny", "bert", "opt", "llama", "opt2048_g8", "llama4096_g8", "opt2048_g8_f32",
             "llama4096_g8_f32"], steps=max(5, min(args.steps, 10)))
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(cfg, lora=args.lora)
        except Exception as ex:  # oracle build failure must not hide the GPU number
            out["cpu_baseline"] = {"error": str(ex)}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

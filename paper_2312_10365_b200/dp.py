"""Token-sharded data parallelism for the routed FFN.

Every token's routing, bucketing, forward and grad-input depend only on that
token and the replicated weights ("each block ... can compute some output
results without synchronizing with the other blocks"; the FFN
treats batch x sequence as independent tokens).  So rank r owns
a contiguous token shard and the only exchange is one SUM all-reduce of the
fp32 weight gradients dw1 | dw2 | dw_r (reading c16: SUM over ranks = the
full-batch gradient of the summed loss; any mean is left to the caller).

The gradients live in ONE flat fp32 buffer so the exchange is a single NCCL
all-reduce (over NVLink/NVSwitch on a B200 node) with no packing copies.

Load-balancing loss (desc.balance_weight = lambda): each rank's
backward differentiates lambda * L_r, the loss of ITS shard's routing
statistics (f_g, pbar_g over its T_r tokens), so the SUM all-reduce yields the
gradient of sum_r lambda * L_r -- a per-shard balance loss, the usual
data-parallel reading of a Switch-style auxiliary loss; it is not the loss of
the global batch's statistics (that would need the per-block counts and
softmax sums all-reduced before the backward).  A caller wanting the mean over
shards passes lambda / world.  tests/test_dp_gloo.py pins this semantics.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(T_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range [t0, t1) of `rank` (sizes differ by at most 1)."""
    base, rem = divmod(T_global, world)
    t0 = rank * base + min(rank, rem)
    return t0, t0 + base + (1 if rank < rem else 0)


class FlatGrads:
    """dw1, dw2, dw_r as views of one contiguous fp32 buffer."""

    def __init__(self, shapes: dict, device="cuda"):
        n = sum(int(torch.Size(s).numel()) for s in shapes.values())
        self.flat = torch.empty(n, dtype=torch.float32, device=device)
        self.views = {}
        off = 0
        for name, s in shapes.items():
            k = int(torch.Size(s).numel())
            self.views[name] = self.flat[off:off + k].view(s)
            off += k

    def __getitem__(self, name):
        return self.views[name]


def attach_flat_grads(ffn, device="cuda") -> FlatGrads:
    """Re-point a RoutedFFN's dw1/dw2/dw_r (a RoutedLoRAFFN's LoRA factor
    gradients db1/dc1/db2/dc2 and dw_r: W is frozen) at views of one flat buffer."""
    if hasattr(ffn, "grads"):  # LoRA-wrapped: the trained tensors only
        fg = FlatGrads({**{n: tuple(g.shape) for n, g in ffn.grads.items()},
                        "dw_r": tuple(ffn.dw_r.shape)}, device)
        ffn.grads = {n: fg[n] for n in ffn.grads}
        ffn.dw_r = fg["dw_r"]
        return fg
    fg = FlatGrads({"dw1": tuple(ffn.dw1.shape), "dw2": tuple(ffn.dw2.shape),
                    "dw_r": tuple(ffn.dw_r.shape)}, device)
    ffn.dw1, ffn.dw2, ffn.dw_r = fg["dw1"], fg["dw2"], fg["dw_r"]
    return fg


def allreduce_grads(fg: FlatGrads, group=None, async_op: bool = False):
    """SUM all-reduce of the flat gradient buffer (no-op on a single process)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(fg.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


class OverlappedAllReduce:
    """SUM all-reduce of the flat gradients that starts, on its own stream, at
    the event spt_ffn_backward records once dw1/dw2/dw_r are final, so it runs
    concurrently with the grad-input kernels of the same backward call."""

    def __init__(self, fg: FlatGrads, group=None):
        self.fg, self.group = fg, group
        self.event = torch.cuda.Event()
        self.stream = torch.cuda.Stream()
        self.active = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1

    def launch(self):
        """Call right after spt_ffn_backward(..., dw_event=self.event)."""
        if not self.active:
            return
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(self.event)
            dist.all_reduce(self.fg.flat, op=dist.ReduceOp.SUM, group=self.group)

    def wait(self, stream=None):
        """Make `stream` (default: current) wait for the all-reduce."""
        if self.active:
            (stream or torch.cuda.current_stream()).wait_stream(self.stream)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device timing is reported as the max over ranks)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

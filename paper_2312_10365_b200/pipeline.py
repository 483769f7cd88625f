"""Host-buffer driver for the routed FFN: steps on token batches that live in
(pinned) host memory, with the copies overlapped with the kernels.

Step i runs route -> forward -> backward (+ optional gradient all-reduce) on a
compute stream while the H2D copy of step i+1's inputs (x, dy) and the D2H copy
of step i-1's outputs (y, dx) run on two copy streams (PCIe is full duplex).
Device inputs and outputs are double-buffered; CUDA events order the streams.
Only argument marshalling and stream/event plumbing live here; every step of the
routed FFN runs in libspt_ffn.so.
"""
from __future__ import annotations

import torch

from .ffn import RoutedFFN


class HostStepPipeline:
    def __init__(self, ffn: RoutedFFN, w1, w2, w_r, grad_hook=None, lora=None):
        self.ffn, self.w1, self.w2, self.w_r = ffn, w1, w2, w_r
        self.lora = lora  # LoRA factors of a RoutedLoRAFFN, else None
        self.grad_hook = grad_hook  # called on the compute stream after backward (e.g. all-reduce)
        T, d, dt = ffn.T, ffn.d, ffn.dtype
        dev = w1.device
        self.x = [torch.empty(T, d, dtype=dt, device=dev) for _ in range(2)]
        self.dy = [torch.empty(T, d, dtype=dt, device=dev) for _ in range(2)]
        self.y = [torch.empty(T, d, dtype=dt, device=dev) for _ in range(2)]
        self.dx = [torch.empty(T, d, dtype=dt, device=dev) for _ in range(2)]
        self.s_h2d, self.s_comp, self.s_d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
        ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.h2d_done, self.comp_done, self.d2h_done = ev(), ev(), ev()
        self.started = [False, False]

    def bytes_per_step(self) -> tuple[int, int]:
        nb = self.x[0].numel() * self.x[0].element_size()
        return 2 * nb, 2 * nb  # H2D x, dy ; D2H y, dx

    def step(self, i: int, x_host, dy_host, y_host, dx_host):
        """Enqueue step i (non-blocking).  Host tensors must be pinned."""
        b = i & 1
        f = self.ffn
        with torch.cuda.stream(self.s_h2d):
            if self.started[b]:
                self.s_h2d.wait_event(self.comp_done[b])      # step i-2 done reading x[b]
            self.x[b].copy_(x_host, non_blocking=True)
            self.dy[b].copy_(dy_host, non_blocking=True)
            self.h2d_done[b].record(self.s_h2d)
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(self.h2d_done[b])
            if self.started[b]:
                self.s_comp.wait_event(self.d2h_done[b])      # step i-2's y[b], dx[b] copied out
            f.y, f.dx = self.y[b], self.dx[b]
            f.route(self.x[b], self.w_r, stream=self.s_comp)
            if self.lora is None:
                f.forward(self.x[b], self.w1, self.w2, stream=self.s_comp)
                f.backward(self.x[b], self.w1, self.w2, self.w_r, self.dy[b], stream=self.s_comp)
            else:
                f.forward(self.x[b], self.w1, self.w2, self.lora, stream=self.s_comp)
                f.backward(self.x[b], self.w1, self.w2, self.w_r, self.lora, self.dy[b],
                           stream=self.s_comp)
            if self.grad_hook is not None:
                self.grad_hook()
            self.comp_done[b].record(self.s_comp)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(self.comp_done[b])
            y_host.copy_(self.y[b], non_blocking=True)
            dx_host.copy_(self.dx[b], non_blocking=True)
            self.d2h_done[b].record(self.s_d2h)
        self.started[b] = True

    def synchronize(self):
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.synchronize()

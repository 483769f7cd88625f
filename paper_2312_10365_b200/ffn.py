"""Thin Python binding of the routed-FFN C ABI (include/spt_ffn.h).

Same names as the C entry points; argument marshalling only (torch tensors ->
device pointers, current CUDA stream).  Every step of the path runs in
libspt_ffn.so's sm_100a kernels.  PyTorch supplies device memory and streams.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L

_DT = {torch.float32: L.SPT_F32, torch.bfloat16: L.SPT_BF16}


def make_desc(T: int, d: int, D: int, G: int, k: int, dtype: torch.dtype, act: int,
              gate: int = L.SPT_GATE_SIGMOID, balance_weight: float = 0.0,
              deterministic: bool = False) -> L.spt_ffn_desc:
    """balance_weight = lambda of the load-balancing loss (0 = off; spt_ffn_balance_loss);
    deterministic = SPT_FFN_DETERMINISTIC (bitwise-reproducible ascending-block k-way sums)."""
    if dtype not in _DT:
        raise ValueError(f"unsupported dtype {dtype}")
    return L.spt_ffn_desc(int(T), int(d), int(D), int(G), int(k), _DT[dtype], int(act), int(gate),
                          float(balance_weight), L.SPT_FFN_DETERMINISTIC if deterministic else 0)


def spt_ffn_sizes(desc: L.spt_ffn_desc) -> tuple[int, int]:
    """(stash_bytes, workspace_bytes) for ``desc``."""
    s, w = ctypes.c_size_t(), ctypes.c_size_t()
    L.check("spt_ffn_sizes", L.lib().spt_ffn_sizes(ctypes.byref(desc), ctypes.byref(s), ctypes.byref(w)))
    return s.value, w.value


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libspt_ffn takes device tensors only")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


@dataclass
class RouteBuffers:
    """Device buffers of spt_route_buf (caller-owned)."""
    logits: torch.Tensor        # [T, G] f32
    topk_idx: torch.Tensor      # [T, k] i32
    topk_gate: torch.Tensor     # [T, k] f32
    block_offsets: torch.Tensor # [G+1] i32
    bucket_token: torch.Tensor  # [T*k] i32
    bucket_gate: torch.Tensor   # [T*k] f32
    pair_slot: torch.Tensor     # [T*k] i32
    tile_offsets: torch.Tensor  # [G+1] i32

    @staticmethod
    def empty(T: int, G: int, k: int, device="cuda") -> "RouteBuffers":
        f, i = dict(dtype=torch.float32, device=device), dict(dtype=torch.int32, device=device)
        return RouteBuffers(torch.empty(T, G, **f), torch.empty(T, k, **i), torch.empty(T, k, **f),
                            torch.empty(G + 1, **i), torch.empty(T * k, **i), torch.empty(T * k, **f),
                            torch.empty(T * k, **i), torch.empty(G + 1, **i))

    def as_c(self) -> L.spt_route_buf:
        return L.spt_route_buf(*[self.__dict__[n].data_ptr() for n, _ in L.spt_route_buf._fields_])


def spt_ffn_route(desc, x, w_r, route: RouteBuffers, ws: torch.Tensor, flags: int = 0, stream=None):
    rb = route.as_c()
    L.check("spt_ffn_route", L.lib().spt_ffn_route(
        ctypes.byref(desc), _p(x), _p(w_r), flags, ctypes.byref(rb), _p(ws), ws.numel() * ws.element_size(),
        _stream(stream)))


def spt_ffn_forward(desc, x, w1, w2, route: RouteBuffers, y, stash, ws, stream=None):
    rb = route.as_c()
    L.check("spt_ffn_forward", L.lib().spt_ffn_forward(
        ctypes.byref(desc), _p(x), _p(w1), _p(w2), ctypes.byref(rb), _p(y), _p(stash), _p(ws),
        ws.numel() * ws.element_size(), _stream(stream)))


def spt_ffn_balance_loss(desc, route: RouteBuffers, loss: torch.Tensor, ws, stream=None):
    """L = G sum_g f_g pbar_g of the routing in ``route`` into the 1-element
    float32 device tensor ``loss`` (reading c18)."""
    rb = route.as_c()
    L.check("spt_ffn_balance_loss", L.lib().spt_ffn_balance_loss(
        ctypes.byref(desc), ctypes.byref(rb), _p(loss), _p(ws), ws.numel() * ws.element_size(),
        _stream(stream)))


def spt_ffn_backward(desc, x, w1, w2, w_r, route: RouteBuffers, stash, dy, dx, dw1, dw2, dw_r,
                     ws, dgate=None, flags: int = 0, stream=None, dw_event=None):
    """dw_event: optional torch.cuda.Event recorded once dw1/dw2/dw_r are final
    (before dx is computed) -- start a gradient all-reduce there."""
    rb = route.as_c()
    ev = None if dw_event is None else ctypes.c_void_p(dw_event.cuda_event)
    L.check("spt_ffn_backward", L.lib().spt_ffn_backward(
        ctypes.byref(desc), _p(x), _p(w1), _p(w2), _p(w_r), ctypes.byref(rb), _p(stash), _p(dy), _p(dx),
        _p(dw1), _p(dw2), _p(dw_r), _p(dgate), flags, _p(ws), ws.numel() * ws.element_size(), ev,
        _stream(stream)))


def spt_ffn_lora_sizes(desc: L.spt_ffn_desc, rank: int) -> tuple[int, int]:
    """(stash_bytes, workspace_bytes) of the LoRA-wrapped calls (ABI 3)."""
    s, w = ctypes.c_size_t(), ctypes.c_size_t()
    L.check("spt_ffn_lora_sizes", L.lib().spt_ffn_lora_sizes(ctypes.byref(desc), int(rank),
                                                              ctypes.byref(s), ctypes.byref(w)))
    return s.value, w.value


def _lora_c(rank, b1, c1, b2, c2) -> L.spt_lora:
    return L.spt_lora(int(rank), *[_p(t) for t in (b1, c1, b2, c2)])


def spt_ffn_lora_forward(desc, x, w1, w2, lora: dict, route: RouteBuffers, y, stash, ws, stream=None):
    """LoRA-wrapped routed forward (include/spt_ffn.h; PAPER.md:159 on fc1/fc2).
    lora: {"b1", "c1", "b2", "c2"} device tensors; the rank is c2.shape[0]."""
    rb = route.as_c()
    lc = _lora_c(lora["c2"].shape[0], lora["b1"], lora["c1"], lora["b2"], lora["c2"])
    L.check("spt_ffn_lora_forward", L.lib().spt_ffn_lora_forward(
        ctypes.byref(desc), _p(x), _p(w1), _p(w2), ctypes.byref(lc), ctypes.byref(rb), _p(y),
        _p(stash), _p(ws), ws.numel() * ws.element_size(), _stream(stream)))


def spt_ffn_lora_backward(desc, x, w1, w2, w_r, lora: dict, route: RouteBuffers, stash, dy, dx,
                          grads: dict, dw_r, ws, dgate=None, flags: int = 0, stream=None,
                          grad_event=None):
    """Backward of spt_ffn_lora_forward (W frozen): dx, grads {"db1", "dc1", "db2",
    "dc2"} (fp32), dw_r; grad_event recorded once every gradient is final."""
    rb = route.as_c()
    lc = _lora_c(lora["c2"].shape[0], lora["b1"], lora["c1"], lora["b2"], lora["c2"])
    gc = L.spt_lora_grads(*[_p(grads[n]) for n in ("db1", "dc1", "db2", "dc2")])
    ev = None if grad_event is None else ctypes.c_void_p(grad_event.cuda_event)
    L.check("spt_ffn_lora_backward", L.lib().spt_ffn_lora_backward(
        ctypes.byref(desc), _p(x), _p(w1), _p(w2), _p(w_r), ctypes.byref(lc), ctypes.byref(rb),
        _p(stash), _p(dy), _p(dx), ctypes.byref(gc), _p(dw_r), _p(dgate), flags, _p(ws),
        ws.numel() * ws.element_size(), ev, _stream(stream)))


def spt_mha_topl(codes_q, codes_k, top_l: int, causal: bool = False, out=None, stream=None,
                 n_codewords: int = 256):
    """Sparse-MHA top-L selection (ABI 4; Alg. 3 over PQ codes, Eq. 3).
    codes_q [H, n_q, M], codes_k [H, n_k, M] uint8 device tensors with every code
    < n_codewords (E; the paper's 16 enables the packed path); returns
    indices [H, n_q, L] int32 (-1 = fewer than L candidates, causal rows)."""
    H, nq, M = codes_q.shape
    nk = codes_k.shape[1]
    if codes_q.dtype != torch.uint8 or codes_k.dtype != torch.uint8:
        raise ValueError("codes must be uint8")
    if codes_k.shape[0] != H or codes_k.shape[2] != M:
        raise ValueError("codes_q / codes_k disagree on heads or codebooks")
    if out is None:
        out = torch.empty(H, nq, int(top_l), dtype=torch.int32, device=codes_q.device)
    d = L.spt_topl_desc(int(H), int(nq), int(nk), int(M), int(n_codewords), int(top_l),
                        1 if causal else 0)
    L.check("spt_mha_topl", L.lib().spt_mha_topl(ctypes.byref(d), _p(codes_q), _p(codes_k), _p(out),
                                                 _stream(stream)))
    return out


def spt_status_string(code: int) -> str:
    return L.status_string(code)


def launch_count() -> int:
    return int(L.lib().spt_ffn_launch_count())


def profile_enable(on: bool = True) -> None:
    L.check("spt_ffn_profile_enable", L.lib().spt_ffn_profile_enable(1 if on else 0))


def profile_read() -> dict:
    """{kernel name: (launches, total_ms)} since profile_enable / the last read."""
    buf = ctypes.create_string_buffer(1 << 16)
    n = L.lib().spt_ffn_profile_read(buf, len(buf))
    if n < 0:
        raise RuntimeError("spt_ffn_profile_read failed")
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


class RoutedFFN:
    """Buffers for one routed-FFN layer shape (a convenience owner of memory;
    the three methods are the ABI calls)."""

    def __init__(self, T, d, D, G, k, dtype, act, gate=L.SPT_GATE_SIGMOID, device="cuda",
                 balance_weight=0.0, deterministic=False):
        self.desc = make_desc(T, d, D, G, k, dtype, act, gate, balance_weight, deterministic)
        self.T, self.d, self.D, self.G, self.k = T, d, D, G, k
        self.dtype, self.act, self.gate = dtype, act, gate
        self.mp = 2 if act == L.SPT_ACT_SWIGLU else 1
        stash_b, ws_b = spt_ffn_sizes(self.desc)
        self.stash = torch.empty(max(stash_b, 16), dtype=torch.uint8, device=device)
        self.ws = torch.empty(max(ws_b, 16), dtype=torch.uint8, device=device)
        self.route_buf = RouteBuffers.empty(T, G, k, device)
        self.y = torch.empty(T, d, dtype=dtype, device=device)
        self.dx = torch.empty(T, d, dtype=dtype, device=device)
        w1_shape = (2, D, d) if self.mp == 2 else (D, d)
        self.dw1 = torch.empty(w1_shape, dtype=torch.float32, device=device)
        self.dw2 = torch.empty(D, d, dtype=torch.float32, device=device)
        self.dw_r = torch.empty(G, d, dtype=torch.float32, device=device)
        self.dgate = torch.empty(T, k, dtype=torch.float32, device=device)
        self.loss_lb = torch.zeros(1, dtype=torch.float32, device=device)

    def route(self, x, w_r, flags=0, stream=None):
        spt_ffn_route(self.desc, x, w_r, self.route_buf, self.ws, flags, stream)
        return self.route_buf

    def balance_loss(self, stream=None):
        """Load-balancing loss of the current routing (device scalar)."""
        spt_ffn_balance_loss(self.desc, self.route_buf, self.loss_lb, self.ws, stream)
        return self.loss_lb

    def forward(self, x, w1, w2, stream=None):
        spt_ffn_forward(self.desc, x, w1, w2, self.route_buf, self.y, self.stash, self.ws, stream)
        return self.y

    def backward(self, x, w1, w2, w_r, dy, flags=0, want_dgate=False, stream=None, dw_event=None):
        spt_ffn_backward(self.desc, x, w1, w2, w_r, self.route_buf, self.stash, dy, self.dx, self.dw1,
                         self.dw2, self.dw_r, self.ws, self.dgate if want_dgate else None, flags, stream,
                         dw_event)
        return self.dx, self.dw1, self.dw2, self.dw_r


class RoutedLoRAFFN(RoutedFFN):
    """Buffers for the LoRA-wrapped routed FFN (ABI 3): W_I, W_O
    frozen, rank-``rank`` factors of both projections trained."""

    def __init__(self, T, d, D, G, k, dtype, act, rank, gate=L.SPT_GATE_SIGMOID, device="cuda",
                 balance_weight=0.0):
        self.desc = make_desc(T, d, D, G, k, dtype, act, gate, balance_weight)
        self.T, self.d, self.D, self.G, self.k, self.rank = T, d, D, G, k, rank
        self.dtype, self.act, self.gate = dtype, act, gate
        self.mp = 2 if act == L.SPT_ACT_SWIGLU else 1
        stash_b, ws_b = spt_ffn_lora_sizes(self.desc, rank)
        self.stash = torch.empty(max(stash_b, 16), dtype=torch.uint8, device=device)
        self.ws = torch.empty(max(ws_b, 16), dtype=torch.uint8, device=device)
        self.route_buf = RouteBuffers.empty(T, G, k, device)
        self.y = torch.empty(T, d, dtype=dtype, device=device)
        self.dx = torch.empty(T, d, dtype=dtype, device=device)
        lead = (2,) if self.mp == 2 else ()
        f = dict(dtype=torch.float32, device=device)
        self.grads = {"db1": torch.empty(lead + (rank, d), **f), "dc1": torch.empty(lead + (D, rank), **f),
                      "db2": torch.empty(D, rank, **f), "dc2": torch.empty(rank, d, **f)}
        self.dw_r = torch.empty(G, d, **f)
        self.dgate = torch.empty(T, k, **f)
        self.loss_lb = torch.zeros(1, **f)

    def forward(self, x, w1, w2, lora, stream=None):
        spt_ffn_lora_forward(self.desc, x, w1, w2, lora, self.route_buf, self.y, self.stash, self.ws,
                             stream)
        return self.y

    def backward(self, x, w1, w2, w_r, lora, dy, flags=0, want_dgate=False, stream=None,
                 grad_event=None):
        spt_ffn_lora_backward(self.desc, x, w1, w2, w_r, lora, self.route_buf, self.stash, dy, self.dx,
                              self.grads, self.dw_r, self.ws, self.dgate if want_dgate else None, flags,
                              stream, grad_event)
        return self.dx, self.grads, self.dw_r

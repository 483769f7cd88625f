"""The C ABI library loads, exports every symbol include/spt_ffn.h declares, and
validates arguments on the host (CPU-only: no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "spt_ffn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spt_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2312_10365_b200 import _lib
    L = _lib.lib()
    decl = _declared_symbols()
    assert set(decl) == set(_lib.EXPORTED), decl
    for name in decl:
        assert hasattr(L, name), name
    assert L.spt_ffn_abi_version() == 5


def test_status_strings():
    from paper_2312_10365_b200 import _lib
    assert _lib.status_string(0) == "SPT_OK"
    assert _lib.status_string(3) == "SPT_ERR_WORKSPACE_TOO_SMALL"
    assert _lib.status_string(99) == "SPT_ERR_UNKNOWN"


def _desc(**kw):
    import torch
    from paper_2312_10365_b200 import make_desc
    a = dict(T=256, d=128, D=512, G=8, k=2, dtype=torch.float32, act=0, gate=0)
    a.update(kw)
    return make_desc(**a)


@pytest.mark.parametrize("G", [129, 200, 256])
def test_bf16_wide_router_supported(G):
    """Reading c25: G up to 256 on the bf16 path (router N = G padded to 16,
    dW_R in two 128-block M halves); sizes grow with G."""
    import torch
    from paper_2312_10365_b200 import spt_ffn_sizes
    s, w = spt_ffn_sizes(_desc(dtype=torch.bfloat16, d=256, G=G, D=G * 64, k=8))
    s1, w1 = spt_ffn_sizes(_desc(dtype=torch.bfloat16, d=256, G=128, D=128 * 64, k=8))
    assert s > s1 > 0 and w > w1 > 0


def test_sizes_valid_and_monotone():
    from paper_2312_10365_b200 import spt_ffn_sizes
    s1, w1 = spt_ffn_sizes(_desc())
    s2, w2 = spt_ffn_sizes(_desc(T=512))
    assert s1 > 0 and w1 > 0 and s2 > s1 and w2 > w1
    s0, w0 = spt_ffn_sizes(_desc(T=0))
    assert s0 >= 0 and w0 >= 0


@pytest.mark.parametrize("kw,code", [
    (dict(k=9), 1),            # k > G
    (dict(k=0), 1),
    (dict(D=500), 1),          # D % G != 0
    (dict(T=-1), 1),
    (dict(d=0), 1),
    (dict(act=7), 1),
    (dict(gate=5), 1),
    (dict(G=512, D=512 * 16, k=2), 2),   # G > 256
    (dict(d=96), 2),                     # d % 64
    (dict(D=8 * 24), 2),                 # bw = 24, not a multiple of 16
])
def test_invalid_descriptors(kw, code):
    from paper_2312_10365_b200 import _lib, spt_ffn_sizes
    with pytest.raises(_lib.SptError) as e:
        spt_ffn_sizes(_desc(**kw))
    assert e.value.code == code


def test_null_pointers_rejected_before_any_launch():
    from paper_2312_10365_b200 import _lib
    L = _lib.lib()
    d = _desc()
    rb = _lib.spt_route_buf()
    assert L.spt_ffn_route(ctypes.byref(d), None, None, 0, ctypes.byref(rb), None, 0, None) == 1
    assert L.spt_ffn_forward(ctypes.byref(d), None, None, None, ctypes.byref(rb), None, None,
                             None, 0, None) == 1
    assert L.spt_ffn_backward(ctypes.byref(d), *([None] * 4), ctypes.byref(rb), *([None] * 7),
                              0, None, 0, None, None) == 1
    s = ctypes.c_size_t()
    assert L.spt_ffn_sizes(None, ctypes.byref(s), ctypes.byref(s)) == 1
    assert L.spt_ffn_sizes(ctypes.byref(d), None, ctypes.byref(s)) == 1


def test_workspace_too_small_rejected():
    from paper_2312_10365_b200 import _lib
    L = _lib.lib()
    d = _desc()
    fake = ctypes.c_void_p(16)  # never dereferenced: size check precedes any launch
    rb = _lib.spt_route_buf(*([16] * 8))
    assert L.spt_ffn_route(ctypes.byref(d), fake, fake, 0, ctypes.byref(rb), fake, 1, None) == 3


def test_desc_layout_and_balance_weight_validation():
    """ABI 2: spt_ffn_desc carries balance_weight (lambda >= 0, finite); the
    workspace grows by the dense router-term buffer only when lambda != 0."""
    import ctypes
    import torch
    from paper_2312_10365_b200 import _lib, spt_ffn_sizes
    assert ctypes.sizeof(_lib.spt_ffn_desc) == 48  # ABI 5: + uint32 flags (padded)
    for bad in (-1.0, float("nan"), float("inf")):
        d = _desc(balance_weight=bad)
        s, w = ctypes.c_size_t(), ctypes.c_size_t()
        assert _lib.lib().spt_ffn_sizes(ctypes.byref(d), ctypes.byref(s), ctypes.byref(w)) == 1
    _, w0 = spt_ffn_sizes(_desc(dtype=torch.bfloat16))
    _, w1 = spt_ffn_sizes(_desc(dtype=torch.bfloat16, balance_weight=0.01))
    assert w1 - w0 == 256 * 128 * 2, w1 - w0   # the dense [T, d] bf16 router term of dx
    # fp32: without the balance gradient the tensor-core (split) path runs and its
    # workspace carries the bf16 hi | lo copies of x, dy and the weights; with it,
    # the SIMT path (f32 [T, G] router term, no copies)
    _, f0 = spt_ffn_sizes(_desc(dtype=torch.float32))
    _, f1 = spt_ffn_sizes(_desc(dtype=torch.float32, balance_weight=0.01))
    assert f0 > f1, (f0, f1)


def test_desc_flags():
    """ABI 5: desc.flags -- unknown bits are rejected; SPT_FFN_DETERMINISTIC is
    accepted and changes nothing (every path sums in ascending block order)."""
    import ctypes
    import torch
    from paper_2312_10365_b200 import _lib, spt_ffn_sizes
    for bad in (2, 0x80000000):
        d = _desc(dtype=torch.bfloat16)
        d.flags = bad
        s, w = ctypes.c_size_t(), ctypes.c_size_t()
        assert _lib.lib().spt_ffn_sizes(ctypes.byref(d), ctypes.byref(s), ctypes.byref(w)) == 1
    for dt in (torch.float32, torch.bfloat16):
        f0, f1 = _desc(dtype=dt), _desc(dtype=dt)
        f1.flags = _lib.SPT_FFN_DETERMINISTIC
        assert spt_ffn_sizes(f0) == spt_ffn_sizes(f1)


# ------------------------------------------------------------ LoRA (ABI 3)
def test_lora_sizes_extend_plain_sizes():
    import torch
    from paper_2312_10365_b200 import spt_ffn_lora_sizes, spt_ffn_sizes
    d = _desc(dtype=torch.bfloat16, d=256, D=1024, G=8, k=2)
    s, w = spt_ffn_sizes(d)
    ls, lw = spt_ffn_lora_sizes(d, 16)
    assert ls > s and lw > w
    ls2, lw2 = spt_ffn_lora_sizes(d, 32)
    assert ls2 >= ls and lw2 > lw


@pytest.mark.parametrize("kw,rank,code", [
    (dict(), 16, 2),                                    # fp32: tcgen05 path only
    (dict(dtype="bf16"), 0, 1),                         # rank < 1
    (dict(dtype="bf16"), 65, 2),                        # m' r > 64
    (dict(dtype="bf16", act=2, D=1024, G=8), 33, 2),    # SwiGLU: 2 r > 64
    (dict(dtype="bf16", k=9), 16, 1),                   # bad descriptor
])
def test_lora_invalid_arguments(kw, rank, code):
    import torch
    from paper_2312_10365_b200 import _lib, spt_ffn_lora_sizes
    if kw.get("dtype") == "bf16":
        kw = dict(kw, dtype=torch.bfloat16)
    with pytest.raises(_lib.SptError) as e:
        spt_ffn_lora_sizes(_desc(**kw), rank)
    assert e.value.code == code


def test_lora_null_pointers_rejected_before_any_launch():
    import torch
    from paper_2312_10365_b200 import _lib
    L = _lib.lib()
    d = _desc(dtype=torch.bfloat16)
    rb = _lib.spt_route_buf()
    lo = _lib.spt_lora(16, None, None, None, None)
    gr = _lib.spt_lora_grads()
    assert L.spt_ffn_lora_forward(ctypes.byref(d), None, None, None, ctypes.byref(lo),
                                  ctypes.byref(rb), None, None, None, 0, None) == 1
    assert L.spt_ffn_lora_forward(ctypes.byref(d), None, None, None, None, ctypes.byref(rb), None,
                                  None, None, 0, None) == 1
    assert L.spt_ffn_lora_backward(ctypes.byref(d), *([None] * 4), ctypes.byref(lo), ctypes.byref(rb),
                                   None, None, None, ctypes.byref(gr), None, None, 0, None, 0, None,
                                   None) == 1


# ------------------------------------------------------------ top-L (ABI 4)
@pytest.mark.parametrize("kw", [dict(n_codebooks=0), dict(n_codebooks=32), dict(top_l=0),
                                dict(n_heads=-1), dict(n_q=-2), dict(causal=2),
                                dict(n_codewords=0), dict(n_codewords=257)])
def test_topl_invalid_arguments(kw):
    from paper_2312_10365_b200 import _lib
    a = dict(n_heads=2, n_q=8, n_k=8, n_codebooks=8, n_codewords=16, top_l=2, causal=0)
    a.update(kw)
    d = _lib.spt_topl_desc(**a)
    dummy = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    assert _lib.lib().spt_mha_topl(ctypes.byref(d), dummy, dummy, dummy, None) == 1


def test_topl_null_and_unsupported():
    from paper_2312_10365_b200 import _lib
    L = _lib.lib()
    d = _lib.spt_topl_desc(2, 8, 8, 8, 16, 2, 0)
    assert L.spt_mha_topl(ctypes.byref(d), None, None, None, None) == 1
    assert L.spt_mha_topl(None, None, None, None, None) == 1
    big = _lib.spt_topl_desc(1, 8, 20000, 16, 256, 4, 0)  # 20000 keys x 32 B > 227 KB smem
    dummy = ctypes.c_void_p(16)
    assert L.spt_mha_topl(ctypes.byref(big), dummy, dummy, dummy, None) == 2
    # the kernel's 40,960 B of static smem count too: M = 16, E = 16 -> 24 B per key,
    # (227 * 1024 - 40960) / 24 = 7978.67 keys fit
    edge = _lib.spt_topl_desc(1, 8, 7979, 16, 16, 4, 0)
    assert L.spt_mha_topl(ctypes.byref(edge), dummy, dummy, dummy, None) == 2
    edge2 = _lib.spt_topl_desc(1, 8, 8192, 16, 16, 4, 0)
    assert L.spt_mha_topl(ctypes.byref(edge2), dummy, dummy, dummy, None) == 2
    empty = _lib.spt_topl_desc(0, 8, 8, 8, 16, 2, 0)
    assert L.spt_mha_topl(ctypes.byref(empty), None, None, None, None) == 0

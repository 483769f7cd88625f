"""GPU parity of the sparse-MHA top-L selection (ABI 4) against
the Algorithm-3 oracle (oracle/topl.py, pinned in test_oracle_topl.py).

Integer work: indices must match the oracle BIT-EXACTLY (north_star: integer,
byte and index work is bit-exact), including the -1 padding of causal rows.
Small cases are checked against the step-by-step form (alg3_topl), the
BASELINE-shaped ones (seq 512-2048, M = 8 / 16, L = n/8) against the closed form
on sampled heads and a block of queries per head.
"""
import numpy as np
import pytest

import synthetic as S
from oracle import topl as OT

pytestmark = pytest.mark.gpu


def gpu_topl(cq, ck, L, causal=False, E=None):
    """E: codewords per codebook (default: max code + 1 -> the packed path when <= 16)."""
    import torch
    import paper_2312_10365_b200 as P
    a = torch.from_numpy(np.ascontiguousarray(cq, np.uint8)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(ck, np.uint8)).cuda()
    if E is None:
        E = int(max(np.max(cq, initial=0), np.max(ck, initial=0))) + 1
    out = P.spt_mha_topl(a, b, L, causal, n_codewords=E)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("E", [3, 16, 200])   # packed nibbles (E <= 16) and bytes
@pytest.mark.parametrize("M", [1, 3, 4, 8, 13, 16, 31])
@pytest.mark.parametrize("causal", [False, True])
def test_step_by_step_small(M, causal, E):
    rng = np.random.default_rng(M)
    H, n = 2, 77
    hi = 3 if E == 3 else E  # E = 3: heavy ties; 16 / 200: the full code range
    cq = rng.integers(0, hi, (H, n, M)).astype(np.uint8)
    ck = cq if causal else rng.integers(0, hi, (H, n, M)).astype(np.uint8)
    if E == 200:  # bytes path: also put equal codes where nibbles would alias (x vs x + 16)
        cq[..., 0] = 17
        if not causal:
            ck[..., 0] = rng.choice([1, 17], size=ck.shape[:2])
    for L in (1, 2, 9, 40, 100):
        got = gpu_topl(cq, ck, L, causal, E=E)
        for h in range(H):
            ref = OT.alg3_topl(cq[h], ck[h], L, causal)
            assert np.array_equal(got[h], ref), (M, causal, L, h)


@pytest.mark.parametrize("name", ["topl_tiny", "topl_bert", "topl_opt", "topl_llama"])
def test_configs_sampled(name):
    cfg = S.TOPL_CONFIGS[name]
    H = min(cfg.heads, 8)
    cq, ck = S.make_pq_codes(cfg, heads=H)
    if cfg.causal:
        ck = cq.copy()
    got = gpu_topl(cq, ck, cfg.L, cfg.causal)
    rng = np.random.default_rng(3)
    for h in range(H):
        qs = np.sort(rng.choice(cfg.n, size=min(cfg.n, 96), replace=False))
        ref = OT.topl_by_sort(cq[h], ck[h], cfg.L, cfg.causal)
        assert np.array_equal(got[h][qs], ref[qs]), (name, h)


def test_all_equal_codes_overflow():
    """every key in bucket M: first L-1 keys then the last key (c21)."""
    cq = np.zeros((1, 5, 8), np.uint8)
    ck = np.zeros((1, 300, 8), np.uint8)
    got = gpu_topl(cq, ck, 10)
    assert (got[0] == np.array(list(range(9)) + [299])).all()


def test_fewer_keys_than_L():
    rng = np.random.default_rng(0)
    cq = rng.integers(0, 4, (3, 20, 8)).astype(np.uint8)
    ck = rng.integers(0, 4, (3, 6, 8)).astype(np.uint8)
    got = gpu_topl(cq, ck, 10)
    for h in range(3):
        assert np.array_equal(got[h], OT.alg3_topl(cq[h], ck[h], 10))
    assert (got[:, :, 6:] == -1).all()


def test_empty():
    import torch
    import paper_2312_10365_b200 as P
    a = torch.empty(0, 10, 8, dtype=torch.uint8, device="cuda")
    assert P.spt_mha_topl(a, a, 4).shape == (0, 10, 4)
    b = torch.zeros(2, 3, 8, dtype=torch.uint8, device="cuda")
    e = torch.empty(2, 0, 8, dtype=torch.uint8, device="cuda")
    out = P.spt_mha_topl(b, e, 4)
    torch.cuda.synchronize()
    assert (out.cpu().numpy() == -1).all()


def test_long_sequence():
    cfg = S.TOPL_CONFIGS["topl_llama"].with_(n=4096)
    cq, ck = S.make_pq_codes(cfg, heads=2)
    got = gpu_topl(cq, ck, cfg.L)
    qs = np.arange(0, 4096, 97)
    for h in range(2):
        assert np.array_equal(got[h][qs], OT.topl_by_sort(cq[h][qs], ck[h], cfg.L))


def test_deterministic():
    cfg = S.TOPL_CONFIGS["topl_bert"]
    cq, ck = S.make_pq_codes(cfg, heads=16)
    a = gpu_topl(cq, ck, cfg.L)
    b = gpu_topl(cq, ck, cfg.L)
    assert np.array_equal(a, b)


def test_max_keys_at_smem_limit():
    """n_k at the shared-memory edge (dynamic + the kernel's static bucket state
    = 227 KB): runs and matches the oracle on sampled queries."""
    rng = np.random.default_rng(11)
    M, nk, L = 16, 7978, 16
    cq = rng.integers(0, 16, (1, 64, M)).astype(np.uint8)
    ck = rng.integers(0, 16, (1, nk, M)).astype(np.uint8)
    got = gpu_topl(cq, ck, L, E=16)
    for q in (0, 31, 63):
        ref = OT.topl_by_sort(cq[0][q:q + 1], ck[0], L, False)
        assert np.array_equal(got[0][q:q + 1], ref)


def test_out_of_range_codes_do_not_fault():
    """Codes >= E are a caller error with unspecified indices but no fault (header):
    on the packed path each code is masked to its nibble, so a score never exceeds M.
    The next call on the same stream still succeeds and is exact."""
    rng = np.random.default_rng(12)
    M, n, L = 5, 300, 8
    cq = rng.integers(0, 256, (2, n, M)).astype(np.uint8)
    ck = rng.integers(0, 256, (2, n, M)).astype(np.uint8)
    got = gpu_topl(cq, ck, L, E=16)
    assert got.shape == (2, n, L) and np.all((got >= -1) & (got < n))
    ok_q, ok_k = cq & 0x7, ck & 0x7
    got2 = gpu_topl(ok_q, ok_k, L, E=16)
    for h in range(2):
        assert np.array_equal(got2[h], OT.alg3_topl(ok_q[h], ok_k[h], L, False))

"""Pins for the oracle of Algorithm 3 (bucket-sort top-L) -- CPU only.

oracle/topl.py is checked against things other than itself:
  * SPEC's worked examples: indicator([1,2],[1,0]) = 1, self-match
    = M; scores [2,1,0] with L = 2 select the score-2 then the score-1 key;
    L >= n selects every key; a causal row 0 selects exactly key 0;
  * an exact brute-force top-L (Python ``sorted`` on the scores, the library
    routine): the selected keys' score multiset equals the L largest scores,
    min selected score >= max unselected score, indices distinct;
  * Eq. 3 scores against a direct double loop;
  * the step-by-step form against the closed form on random, clustered,
    all-equal and single-codebook inputs, including bucket overflow (c21) and
    causal rows (c23).
"""
import numpy as np
import pytest

import synthetic as S
from oracle import topl as OT


def test_spec_indicator_examples():
    assert OT.indicator([1, 2], [1, 0]) == 1
    c = [3, 1, 4, 1]
    assert OT.indicator(c, c) == 4
    rng = np.random.default_rng(0)
    cq, ck = rng.integers(0, 4, (9, 8)), rng.integers(0, 4, (7, 8))
    s = OT.pq_scores(cq, ck)
    for q in range(9):
        for k in range(7):
            n = 0
            for m in range(8):
                n += int(cq[q, m] == ck[k, m])
            assert s[q, k] == n


def test_spec_select_example():
    cq = np.array([[1, 1]])
    ck = np.array([[1, 1], [1, 0], [0, 0]])      # scores [2, 1, 0]
    assert OT.alg3_topl(cq, ck, 2).tolist() == [[0, 1]]
    assert OT.alg3_topl(cq, ck, 3).tolist() == [[0, 1, 2]]   # L >= n: all keys


def test_causal_row0_selects_key0():
    rng = np.random.default_rng(1)
    c = rng.integers(0, 3, (6, 4))
    out = OT.alg3_topl(c, c, 3, causal=True)
    assert out[0].tolist() == [0, -1, -1]
    for q in range(6):
        row = out[q][out[q] >= 0]
        assert len(row) == min(3, q + 1) and row.max() <= q


def _brute_check(cq, ck, L, out, causal=False):
    s = OT.pq_scores(cq, ck)
    for q in range(len(cq)):
        cand = list(range(min(len(ck), q + 1) if causal else len(ck)))
        sel = [int(k) for k in out[q] if k >= 0]
        assert len(sel) == min(L, len(cand))
        assert len(set(sel)) == len(sel) and all(k in cand for k in sel)
        best = sorted((int(s[q, k]) for k in cand), reverse=True)[:L]
        assert sorted((int(s[q, k]) for k in sel), reverse=True) == best
        rest = [int(s[q, k]) for k in cand if k not in sel]
        if rest and sel:
            assert min(int(s[q, k]) for k in sel) >= max(rest)
        # Alg. 3 emits buckets from score M down (c22)
        sc = [int(s[q, k]) for k in sel]
        assert sc == sorted(sc, reverse=True)


@pytest.mark.parametrize("L", [1, 2, 5, 16, 40])
@pytest.mark.parametrize("causal", [False, True])
def test_exact_top_l_multiset(L, causal):
    rng = np.random.default_rng(L)
    cq = rng.integers(0, 3, (40, 6))
    ck = cq if causal else rng.integers(0, 3, (33, 6))
    out = OT.alg3_topl(cq, ck, L, causal)
    _brute_check(cq, ck, L, out, causal)


def test_overflow_keeps_first_L_minus_1_and_last():
    """c21: 7 keys in one bucket, L = 4 -> slots hold keys 0,1,2 and the last (6)."""
    cq = np.zeros((1, 3), int)
    ck = np.zeros((7, 3), int)
    assert OT.alg3_topl(cq, ck, 4).tolist() == [[0, 1, 2, 6]]
    assert OT.alg3_topl(cq, ck, 1).tolist() == [[6]]


@pytest.mark.parametrize("kind", ["random", "clustered", "equal", "m1"])
@pytest.mark.parametrize("causal", [False, True])
def test_step_by_step_equals_closed_form(kind, causal):
    rng = np.random.default_rng(7)
    if kind == "random":
        cq = rng.integers(0, 16, (64, 8))
        ck = rng.integers(0, 16, (64, 8))
    elif kind == "clustered":
        a, b = S.make_pq_codes(S.TOPL_CONFIGS["topl_tiny"].with_(n=96), heads=1)
        cq, ck = a[0], b[0]
    elif kind == "equal":
        cq = np.ones((20, 4), int)
        ck = np.ones((20, 4), int)
    else:
        cq = rng.integers(0, 2, (50, 1))
        ck = rng.integers(0, 2, (50, 1))
    if causal:
        ck = cq
    for L in (1, 3, 12, 70):
        a = OT.alg3_topl(cq, ck, L, causal)
        assert np.array_equal(a, OT.topl_by_sort(cq, ck, L, causal)), L
        _brute_check(cq, ck, L, a, causal)


def test_synthetic_codes():
    cfg = S.TOPL_CONFIGS["topl_llama"]
    q, k = S.make_pq_codes(cfg, heads=2)
    assert q.shape == (2, cfg.n, 16) and q.dtype == np.uint8 and q.max() < cfg.E
    s = OT.pq_scores(q[0, :64], k[0])
    assert s.min() == 0 and s.max() >= 12       # scores span the range (clustered codes)
    assert cfg.L == 256

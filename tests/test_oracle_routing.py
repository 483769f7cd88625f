"""Pins for the oracle's routing (a2 top-k) and bucketing (a3) -- CPU only.

Each test pins oracle/spt_oracle.c against something other than itself:
the SPEC's worked examples (tests/golden/), a brute-force Python sort, and a
library stable sort (numpy argsort kind="stable").
"""
import json
import os
import struct

import numpy as np
import pytest

import synthetic as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _absbits(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", v))[0] & 0x7FFFFFFF


def brute_topk(logits, k):
    """Definition (PAPER.md:435 + readings c3/c4) via Python's sorted()."""
    out = []
    for row in np.asarray(logits, np.float32):
        order = sorted(range(len(row)), key=lambda b: (-_absbits(float(row[b])), b))
        out.append(sorted(order[:k]))
    return np.array(out, dtype=np.int32).reshape(len(out), k)


@pytest.mark.parametrize("fname", ["spec_route_example.json", "spec_route_all.json"])
def test_golden_spec_examples(orc, fname):
    g = json.load(open(os.path.join(GOLD, fname)))
    got = orc.topk(np.array(g["logits"], np.float32), g["k"])
    assert got.tolist() == g["selected_set"]


def test_k_out_of_range_is_error(orc):
    lg = np.zeros((2, 4), np.float32)
    with pytest.raises(ValueError):
        orc.topk(lg, 5)          # SPEC S:325 "G' > G -> config error"
    with pytest.raises(ValueError):
        orc.topk(lg, 0)


@pytest.mark.parametrize("kind", ["normal", "zipf", "same", "ties", "signed0"])
@pytest.mark.parametrize("G,k", [(8, 1), (8, 2), (8, 8), (32, 8), (86, 22), (5, 3)])
def test_topk_matches_bruteforce(orc, kind, G, k):
    lg = S.make_logits(97, G, k, kind)
    assert np.array_equal(orc.topk(lg, k), brute_topk(lg, k))


def test_topk_special_values(orc):
    inf, nan = np.float32(np.inf), np.float32(np.nan)
    lg = np.array([[1.0, -inf, nan, 2.0, inf, -0.0, 0.0, -nan]], np.float32)
    # NaN bit patterns (0x7fc00000) rank above +Inf (0x7f800000) -- reading c4
    for k in range(1, 9):
        assert np.array_equal(orc.topk(lg, k), brute_topk(lg, k))
    assert orc.topk(lg, 2).tolist() == [[2, 7]]          # both NaNs
    assert orc.topk(lg, 4).tolist() == [[1, 2, 4, 7]]    # then -inf (id 1) before +inf (id 4)
    # +0 / -0 tie -> lower id
    assert orc.topk(np.array([[-0.0, 0.0, -0.0]], np.float32), 1).tolist() == [[0]]


def _bucket_by_stable_sort(topk_idx, G, tile_m):
    """Library routine: numpy's stable argsort of the pairs by block id."""
    T, k = topk_idx.shape
    flat = topk_idx.reshape(-1)                      # pair q = t*k + j, token q // k
    order = np.argsort(flat, kind="stable")          # block-major, token-ascending
    counts = np.bincount(flat, minlength=G)
    bo = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    tiles = (counts + tile_m - 1) // tile_m
    to = np.concatenate([[0], np.cumsum(tiles)]).astype(np.int32)
    bt = (order // k).astype(np.int32)
    ps = np.empty(T * k, np.int32)
    ps[order] = np.arange(T * k, dtype=np.int32)
    return bo, bt, ps, to


@pytest.mark.parametrize("kind", ["normal", "zipf", "same", "ties"])
@pytest.mark.parametrize("T,G,k", [(1, 8, 2), (257, 8, 2), (300, 32, 8), (1000, 86, 22), (129, 4, 4)])
def test_bucket_matches_stable_sort_and_invariants(orc, kind, T, G, k):
    ti = orc.topk(S.make_logits(T, G, k, kind), k)
    r = orc.bucket(ti, G, tile_m=128)
    bo, bt, ps, to = _bucket_by_stable_sort(ti, G, 128)
    assert np.array_equal(r["block_offsets"], bo)
    assert np.array_equal(r["bucket_token"], bt)
    assert np.array_equal(r["pair_slot"], ps)
    assert np.array_equal(r["tile_offsets"], to)
    # invariants (SURVEY §8(c) bucket pin)
    assert r["block_offsets"][G] == T * k
    assert np.all(np.diff(r["block_offsets"]) >= 0)
    assert np.array_equal(np.bincount(r["bucket_token"], minlength=T), np.full(T, k))
    for b in range(G):
        seg = r["bucket_token"][r["block_offsets"][b]:r["block_offsets"][b + 1]]
        assert np.all(np.diff(seg) > 0)             # strictly increasing tokens
    t_of = np.repeat(np.arange(T), k)
    assert np.array_equal(r["bucket_token"][r["pair_slot"]], t_of)
    blk_of_slot = np.searchsorted(r["block_offsets"], r["pair_slot"], side="right") - 1
    assert np.array_equal(blk_of_slot, ti.reshape(-1))


def test_bucket_empty(orc):
    ti = np.zeros((0, 2), np.int32)
    r = orc.bucket(ti, 8)
    assert r["block_offsets"].tolist() == [0] * 9
    assert r["tile_offsets"].tolist() == [0] * 9

"""CPU oracle of SPT's bucket-sort top-L selection (Algorithm 3) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module; it never imports the product.

What it computes (the sparse-MHA selection step, Alg. 2
line 3):
  * PQ codes: every query / key vector is a row of M codeword ids
    t^1..t^M (one per codebook); codes are integers.
  * Eq. 3:  s(q, k) = sum_m I[t^m_q = t^m_k]  in {0..M}.
  * Algorithm 3 "The procedure of top-L selection", per
    query q:
        Ptr <- allocate(M+1) (zeros), Bucket <- allocate((M+1) x L)    line 2
        for key k in C_K (ascending key index):                          line 3
            s <- indicator(c_q, c_k)                                     line 4
            ptr <- Ptr[s]; Bucket[s][ptr] <- k                           lines 5-6
            Ptr[s] <- min(ptr + 1, L - 1)                                line 7
        s <- M, ptr <- 0                                                 line 9
        for i = 0 .. L-1:                                                line 10
            while ptr == len(s): ptr <- 0, s <- s - 1                    lines 11-12
            Indices_q[i] <- Bucket[s][ptr++]                             line 14

Readings (DESIGN.md c20-c23; SPEC S:186-213 takes the same ones):
  c20  line 11 is applied as ``while`` (the paper writes ``if``): retrieval
       "checks the buckets from high index to low index ... and stops when L
       keys are collected"; a literal ``if`` would read an empty
       bucket's unwritten slot.
  c21  capacity: a bucket holds L keys ("capacity of each bucket as L",
       PAPER.md:520) and on overflow the new key overwrites slot L-1 (line 7:
       the write position never passes L-1; "we overwrite an old key with the
       new key").  The readable length len(s) of bucket s is
       min(#keys inserted, L): a bucket yields its first L-1 keys and, when it
       received L or more, its LAST key in slot L-1.  (Reading Ptr itself as the
       readable length would drop slot L-1 and could return a lower-score key
       while a higher-score one exists -- against "the top-L".)
  c22  keys are visited in ascending index (line 3); outputs are ordered by
       bucket (M first) and, within a bucket, by slot.
  c23  causal (decoder) rows: the look-ahead mask of PAPER.md:329 is applied
       before bucketing (keys k > q are not candidates); a row with
       fewer than L candidates is padded with -1 after its candidates.

``alg3_topl`` is the step-by-step form (Python loops; small inputs).
``topl_by_sort`` is the closed form used for larger parity cases (a stable
sort by descending score, each score group cut to its first L-1 keys plus its
last key) -- pinned to ``alg3_topl`` and to an exact brute-force top-L score
multiset in tests/test_oracle_topl.py.  Parity status: pinned.
"""
from __future__ import annotations

import numpy as np


def pq_scores(cq, ck) -> np.ndarray:
    """Eq. 3: s[q, k] = number of codebooks m with cq[q, m] == ck[k, m]  ([nq, nk] int)."""
    cq = np.asarray(cq)
    ck = np.asarray(ck)
    return (cq[:, None, :] == ck[None, :, :]).sum(axis=2)


def indicator(cq_row, ck_row) -> int:
    """Eq. 3 for one query / key pair (Alg. 3 line 4)."""
    return int(sum(1 for a, b in zip(cq_row, ck_row) if a == b))


def alg3_topl(cq, ck, L: int, causal: bool = False) -> np.ndarray:
    """Algorithm 3 step by step (readings c20-c23).  cq [nq, M], ck [nk, M]
    integer codes; returns Indices [nq, L] int32 (-1 = no candidate left)."""
    cq = np.asarray(cq)
    ck = np.asarray(ck)
    nq, M = cq.shape
    nk = ck.shape[0]
    if L < 1:
        raise ValueError("L >= 1")
    out = np.full((nq, L), -1, dtype=np.int32)
    for q in range(nq):                                   # line 1
        Ptr = [0] * (M + 1)                               # line 2
        Cnt = [0] * (M + 1)                               # keys inserted per bucket (c21)
        Bucket = [[-1] * L for _ in range(M + 1)]
        for k in range(nk):                               # line 3
            if causal and k > q:                          # c23: look-ahead mask
                break
            s = indicator(cq[q], ck[k])                   # line 4
            ptr = Ptr[s]                                  # line 5
            Bucket[s][ptr] = k                            # line 6
            Ptr[s] = min(ptr + 1, L - 1)                  # line 7
            Cnt[s] += 1
        s, ptr = M, 0                                     # line 9
        for i in range(L):                                # line 10
            while s >= 0 and ptr == min(Cnt[s], L):       # lines 11-12 (c20: while; c21)
                ptr, s = 0, s - 1
            if s < 0:                                     # fewer than L candidates (c23)
                break
            out[q, i] = Bucket[s][ptr]                    # line 14
            ptr += 1
    return out


def topl_by_sort(cq, ck, L: int, causal: bool = False) -> np.ndarray:
    """Closed form of alg3_topl: keys ordered by (score descending, key
    ascending) -- a stable sort -- with each score group cut to its first L-1
    keys plus, if it has L or more, its last key (c21); first L; -1 padded."""
    s = pq_scores(cq, ck)
    nq, nk = s.shape
    out = np.full((nq, L), -1, dtype=np.int32)
    for q in range(nq):
        cand = np.arange(min(nk, q + 1) if causal else nk)
        sq = s[q, cand]
        picked = []
        for v in range(int(sq.max()) if cand.size else -1, -1, -1):
            grp = cand[sq == v]
            if grp.size >= L:
                grp = np.concatenate([grp[:L - 1], grp[-1:]])
            picked.extend(grp.tolist())
            if len(picked) >= L:
                break
        m = min(L, len(picked))
        out[q, :m] = picked[:m]
    return out

"""Pure-Python loop mini-oracle for tiny inputs (TEST INFRASTRUCTURE).

An independent second implementation of the same definitions as
ckv_oracle.py, written with scalar loops and `math` only (no NumPy linear
algebra), used to pin the NumPy oracle on n <= 64, m <= 16, n_s <= 4, d <= 8.
Definitions: PAPER.md:99 (softmax attention), 428-435 (token score, Eq. 1),
387 (top-k), SURVEY §8(c) Q1-Q9 readings.
"""
from __future__ import annotations

import itertools
import math


def _dot(x, y):
    return sum(a * b for a, b in zip(x, y))


def scores(Qs, Kp, c, G):
    """Returns (a, A) by explicit loops: for every head h and suffix row r, the
    softmax over all prefix keys, accumulated per key token, then summed per chunk."""
    ns, hq, d = len(Qs), len(Qs[0]), len(Qs[0][0])
    n = len(Kp)
    a = [0.0] * n
    for h in range(hq):
        for r in range(ns):
            l = [_dot(Qs[r][h], Kp[i][h // G]) / math.sqrt(d) for i in range(n)]
            mx = max(l)
            e = [math.exp(x - mx) for x in l]
            s = sum(e)
            for i in range(n):
                a[i] += e[i] / s
    m = (n + c - 1) // c
    A = [sum(a[j * c:min((j + 1) * c, n)]) for j in range(m)]
    return a, A


def best_subset(A, k):
    """Brute force: among all k-subsets, the max total score; among those the
    lexicographically smallest sorted index tuple (lowest-index tie-break)."""
    best = None
    for sub in itertools.combinations(range(len(A)), k):
        tot = sum(A[j] for j in sub)
        if best is None or tot > best[0] + 1e-12 * max(1.0, abs(best[0])):
            best = (tot, sub)
    return list(best[1])


def attend(Qs, Ks, Vs, Kp, Vp, tokens, G):
    """O[r][h] = sum over kept prefix tokens and suffix t <= r of softmax(q.k/sqrt(d)) v."""
    ns, hq, d = len(Qs), len(Qs[0]), len(Qs[0][0])
    O = [[[0.0] * d for _ in range(hq)] for _ in range(ns)]
    for r in range(ns):
        for h in range(hq):
            kv = h // G
            keys = [(Kp[i][kv], Vp[i][kv]) for i in tokens] + [(Ks[t][kv], Vs[t][kv]) for t in range(r + 1)]
            l = [_dot(Qs[r][h], kk) / math.sqrt(d) for kk, _ in keys]
            mx = max(l)
            e = [math.exp(x - mx) for x in l]
            s = sum(e)
            for (kk, vv), w in zip(keys, e):
                for x in range(d):
                    O[r][h][x] += w / s * vv[x]
    return O

"""Plain fp64 NumPy oracle of the per-layer Re-Prefill hot path (TEST INFRASTRUCTURE).

Independent of the CUDA path: no shared code, headers, tables or helpers.
Inputs are the exact bf16 (or fp32) values the GPU sees, upcast to float64.

Notation follows PAPER.md: n prefix tokens, chunk size c, m = ceil(n/c)
ContiguousChunks (Def. 2), suffix length n_s, Hq query heads
sharing Hkv KV heads in groups of G = Hq/Hkv (GQA), head dim
d.  Readings of the paper's silent/garbled points are SURVEY.md §8(c) Q1-Q16
(restated in DESIGN.md §2).

Pins (tests/test_oracle_pins.py, tests/test_oracle_brute.py):
  chunk_count/chunk_range   SPEC.md:61-79 worked examples + partition property
  budget_chunks             hand-computed floor rule values (Q7)
  token_scores              closed forms (uniform logits, +50 saturation),
                            conservation sum_i a_i = n_s*Hq, brute force
  chunk_scores              SPEC.md:212 worked example, conservation
  select_topk               SPEC.md:222-224 worked examples, brute-force subset
                            enumeration (m <= 16), nesting, c=1 == np.lexsort
  attention                 k = m equals torch SDPA (fp64) dense causal
                            attention; single-key closed form; brute force
  lse_merge                 split/merge identity vs direct attention
  sharded_reprefill_layer   identity with the unsharded oracle (W = 2, 4, 8)
"""
from __future__ import annotations

import numpy as np

NORM_PREFIX = 0    # Q1 default: softmax over the n prefix keys only
NORM_FULLROW = 1   # Q1 alternative: prefix keys + causal suffix keys


# ---------------------------------------------------------------- geometry
def chunk_count(n: int, c: int) -> int:
    """m = ceil(n / c)  (Def. 2)."""
    if n < 1 or c < 1:
        raise ValueError("n and c must be >= 1")
    return -(-n // c)


def chunk_range(j: int, n: int, c: int) -> tuple[int, int]:
    """Token range [j*c, min((j+1)*c, n)) of 0-based chunk j  (Eq. 1; Q5, Q6)."""
    m = chunk_count(n, c)
    if not 0 <= j < m:
        raise ValueError("chunk index out of range")
    return j * c, min((j + 1) * c, n)


def budget_chunks(n: int, c: int, budget_bp: int) -> int:
    """k = max(1, min(m, floor(budget_bp * n / (10000 * c))))  (Q7: "top-k chunks under
    the token budget", budget ratio PAPER.md:516, in integer basis points)."""
    if not 1 <= budget_bp <= 10000:
        raise ValueError("budget_bp must be in [1, 10000]")
    m = chunk_count(n, c)
    return max(1, min(m, (budget_bp * n) // (10000 * c)))


# ---------------------------------------------------------------- scoring
def _f64(x):
    return np.asarray(x, dtype=np.float64)


def _logsumexp(x: np.ndarray, axis: int) -> np.ndarray:
    mx = np.max(x, axis=axis, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    return np.squeeze(mx, axis) + np.log(np.sum(np.exp(x - mx), axis=axis))


def prefix_logits(Qs, Kp, G: int, kvh: int) -> np.ndarray:
    """l[g, r, i] = q_{r, kvh*G+g} . k_{i, kvh} / sqrt(d)  for one KV head.

    softmax(h_q . h_k) of PAPER.md:99, 429 with the 1/sqrt(d) of the "standard
    attention mechanism" (Q3); query head h uses KV head floor(h/G) (GQA)."""
    Qs, Kp = _f64(Qs), _f64(Kp)
    d = Qs.shape[-1]
    q = Qs[:, kvh * G:(kvh + 1) * G, :].transpose(1, 0, 2)  # [G, n_s, d]
    return (q @ Kp[:, kvh, :].T) / np.sqrt(d)  # [G, n_s, n]


def _suffix_logits(Qs, Ks, G: int, kvh: int) -> np.ndarray:
    """Causal suffix logits [G, n_s, n_s], -inf where t > r  (Q9)."""
    Qs, Ks = _f64(Qs), _f64(Ks)
    d = Qs.shape[-1]
    ns = Qs.shape[0]
    q = Qs[:, kvh * G:(kvh + 1) * G, :].transpose(1, 0, 2)
    l = (q @ Ks[:, kvh, :].T) / np.sqrt(d)
    mask = np.arange(ns)[None, :] > np.arange(ns)[:, None]
    return np.where(mask[None], -np.inf, l)


def row_lse(Qs, Kp, G: int, norm: int = NORM_PREFIX, Ks=None) -> np.ndarray:
    """Lambda[h, r] = log sum_i exp(l[h, r, i]): the softmax normaliser of each
    suffix row over the prefix keys (Q1); FULLROW adds the causal suffix keys."""
    Qs = _f64(Qs)
    ns, hq, _ = Qs.shape
    hkv = hq // G
    lam = np.empty((hq, ns))
    for kvh in range(hkv):
        l = prefix_logits(Qs, Kp, G, kvh)
        lse = _logsumexp(l, axis=-1)
        if norm == NORM_FULLROW:
            lse = np.logaddexp(lse, _logsumexp(_suffix_logits(Qs, Ks, G, kvh), axis=-1))
        lam[kvh * G:(kvh + 1) * G] = lse
    return lam


def token_scores(Qs, Kp, G: int, norm: int = NORM_PREFIX, Ks=None, lam=None):
    """a_i = sum_h sum_r softmax_r(l)[h, r, i]  (column sum of
    h_qk "over the second dimension" read as the query axis (Q2), summed over all
    Hq heads (Q4)).  Returns (a [n], Lambda [Hq, n_s])."""
    Qs = _f64(Qs)
    ns, hq, _ = Qs.shape
    hkv = hq // G
    if lam is None:
        lam = row_lse(Qs, Kp, G, norm, Ks)
    n = np.asarray(Kp).shape[0]
    a = np.zeros(n)
    for kvh in range(hkv):
        l = prefix_logits(Qs, Kp, G, kvh)
        a += np.exp(l - lam[kvh * G:(kvh + 1) * G, :, None]).sum(axis=(0, 1))
    return a, lam


def chunk_scores(a, c: int) -> np.ndarray:
    """A_j = a_{jc} + ... + a_{min((j+1)c, n)-1}  (Eq. 1, PAPER.md:431-435, 0-based; Q5, Q6)."""
    a = _f64(a)
    n = a.shape[0]
    m = chunk_count(n, c)
    return np.array([a[j * c:min((j + 1) * c, n)].sum() for j in range(m)])


# ---------------------------------------------------------------- selection
def select_topk(A, k: int) -> np.ndarray:
    """The k largest A_j, ties to the lower index, returned ascending
    ("identifies the critical tokens"; Q7, Q8)."""
    A = _f64(A)
    m = A.shape[0]
    if not 1 <= k <= m:
        raise ValueError("k out of range")
    order = sorted(range(m), key=lambda j: (-A[j], j))
    return np.array(sorted(order[:k]), dtype=np.int64)


def score_gap(A, k: int) -> float:
    """(A_(k) - A_(k+1)) / A_(k) of the scores sorted descending;
    inf when k = m (no (k+1)-th score), 0 when A_(k) <= 0."""
    A = np.sort(_f64(A))[::-1]
    if not 1 <= k <= A.shape[0]:
        raise ValueError("k out of range")
    if k == A.shape[0]:
        return float("inf")
    if A[k - 1] <= 0:
        return 0.0
    return float((A[k - 1] - A[k]) / A[k - 1])


GAP_GATE = 1e-3      # Q11: relative k/k+1 gap above which the selected set is unique in practice
FLOOR_REL = 1e-30    # Q11: A_(k+1) at or below this share of sum(A) is fp32 underflow noise


def parity_gate(A, k: int, gate: float = GAP_GATE, floor: float = FLOOR_REL) -> bool:
    """True when the top-k set must be reproduced bit-exactly:
    k = m, or gap (A_(k) - A_(k+1)) / A_(k) > gate AND A_(k+1) > floor * sum(A).
    Otherwise several sets are correct (near-ties, or scores at the fp32 underflow floor)."""
    A = _f64(A)
    if k == A.shape[0]:
        return True
    s = np.sort(A)[::-1]
    return bool(score_gap(A, k) > gate and s[k] > floor * A.sum())


def valid_relaxed_set(A, k: int, ids, gate: float = GAP_GATE) -> bool:
    """Q11 relaxed validity of a selected set when parity_gate is False: |ids| = k distinct
    in-range ids, every chosen chunk scores >= A_(k)(1 - gate), and every chunk scoring
    > A_(k)(1 + gate) is chosen -- only true near-ties of the k-th score may differ."""
    A = _f64(A)
    ids = np.asarray(ids, dtype=np.int64)
    m = A.shape[0]
    if ids.shape[0] != k or len(set(ids.tolist())) != k or ids.min() < 0 or ids.max() >= m:
        return False
    Ak = np.sort(A)[::-1][k - 1]
    must = np.nonzero(A > Ak * (1 + gate))[0]
    return bool(np.all(A[ids] >= Ak * (1 - gate)) and set(must.tolist()) <= set(ids.tolist()))


def coverage_ratio(a, b) -> float:
    """|a & b| / |a|  (coverage ratio between index sets)."""
    a, b = set(int(x) for x in a), set(int(x) for x in b)
    if not a:
        raise ValueError("empty set")
    return len(a & b) / len(a)


# ---------------------------------------------------------------- attention
def kept_token_index(sel, n: int, c: int) -> np.ndarray:
    """Prefix token indices of the selected chunks, in ascending order (padding of a
    partial last chunk excluded, Q6)."""
    out = [np.arange(*chunk_range(int(j), n, c)) for j in sel]
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


def attention(Qs, Ks, Vs, Kp, Vp, tokens, G: int, include_suffix: bool = True):
    """Exact softmax attention of every suffix row over the kept prefix tokens
    (all visible) plus the causal suffix t <= r  (PAPER.md:97-99 softmax(q.k).v,
    Def. 1 at PAPER.md:159; north_star step 4; Q9).

    Returns (O [n_s, Hq, d], lse [n_s, Hq]); rows with no key get O = 0, lse = -inf."""
    Qs, Ks, Vs, Kp, Vp = map(_f64, (Qs, Ks, Vs, Kp, Vp))
    ns, hq, d = Qs.shape
    hkv = hq // G
    tokens = np.asarray(tokens, dtype=np.int64)
    O = np.zeros((ns, hq, d))
    lse = np.full((ns, hq), -np.inf)
    for kvh in range(hkv):
        parts_l, parts_v = [], []
        if tokens.size:
            q = Qs[:, kvh * G:(kvh + 1) * G, :].transpose(1, 0, 2)
            parts_l.append((q @ Kp[tokens, kvh, :].T) / np.sqrt(d))
            parts_v.append(Vp[tokens, kvh, :])
        if include_suffix:
            parts_l.append(_suffix_logits(Qs, Ks, G, kvh))
            parts_v.append(Vs[:, kvh, :])
        if not parts_l:
            continue
        l = np.concatenate(parts_l, axis=-1)  # [G, n_s, T]
        v = np.concatenate(parts_v, axis=0)   # [T, d]
        row = _logsumexp(l, axis=-1)          # [G, n_s]
        p = np.exp(l - np.where(np.isfinite(row), row, 0.0)[..., None])
        p = np.where(np.isfinite(row)[..., None], p, 0.0)
        o = p @ v                             # [G, n_s, d]
        O[:, kvh * G:(kvh + 1) * G, :] = o.transpose(1, 0, 2)
        lse[:, kvh * G:(kvh + 1) * G] = row.T
    return O, lse


def lse_merge(parts):
    """Merge normalised partial attentions (O_s, lse_s) over disjoint key sets:
    O = sum_s exp(lse_s - M) O_s / sum_s exp(lse_s - M), lse = M + log sum_s exp(lse_s - M)
    (the exact softmax of PAPER.md:99 split over key subsets)."""
    Os = np.stack([_f64(p[0]) for p in parts])
    ls = np.stack([_f64(p[1]) for p in parts])
    M = np.max(ls, axis=0)
    Mf = np.where(np.isfinite(M), M, 0.0)
    w = np.where(np.isfinite(ls), np.exp(ls - Mf), 0.0)
    den = w.sum(axis=0)
    O = (w[..., None] * Os).sum(axis=0) / np.where(den > 0, den, 1.0)[..., None]
    lse = np.where(den > 0, Mf + np.log(np.where(den > 0, den, 1.0)), -np.inf)
    return O, lse


# ---------------------------------------------------------------- one layer
def reprefill_layer(Qs, Ks, Vs, Kp, Vp, c: int, k: int, G: int, norm: int = NORM_PREFIX,
                    sel=None):
    """One layer of the Re-Prefill hot path:
    score chunks (Eq. 1), select top-k, attend over kept chunks + causal suffix.
    If `sel` is given, the selection step is skipped and attention uses it (Q11 (iii))."""
    a, lam = token_scores(Qs, Kp, G, norm, Ks)
    A = chunk_scores(a, c)
    n = np.asarray(Kp).shape[0]
    if sel is None:
        sel = select_topk(A, k)
    O, lse = attention(Qs, Ks, Vs, Kp, Vp, kept_token_index(sel, n, c), G)
    return {"ids": np.asarray(sel), "out": O, "lse": lse, "A": A, "a": a, "Lambda": lam,
            "gap": score_gap(A, k)}


def shard_chunks(W: int, g: int, m: int, cyclic: bool = False) -> list[int]:
    """Chunk ids owned by shard g of W: contiguous [g*ceil(m/W), min((g+1)*ceil(m/W), m)),
    or cyclic {j : j mod W == g} (the balanced alternative of SURVEY §8(f) NEXT-3), ascending."""
    if cyclic:
        return list(range(g, m, W))
    per = -(-m // W)
    return list(range(min(g * per, m), min((g + 1) * per, m)))


def sharded_reprefill_layer(W: int, Qs, Ks, Vs, Kp, Vp, c: int, k: int, G: int,
                            norm: int = NORM_PREFIX, cyclic: bool = False):
    """Position-sharded form of reprefill_layer, written out step by step:
    shard g owns the chunks shard_chunks(W, g, m, cyclic) and scores the tokens of those chunks.
      1. shard-local Lambda_g = LSE over the shard's keys; 2. global Lambda = LSE_g Lambda_g
      (+ the causal-suffix term on rank W-1 in FULLROW mode);
      3. shard A_j with the global Lambda; 4. local top-min(k, m_g) candidates -> merged top-k;
      5. per-shard attention over owned kept chunks (suffix on rank W-1); 6. LSE merge."""
    Qs_, Kp_ = _f64(Qs), _f64(Kp)
    n = Kp_.shape[0]
    m = chunk_count(n, c)
    shards = [shard_chunks(W, g, m, cyclic) for g in range(W)]
    ns, hq, _ = Qs_.shape
    lam_g = []
    for own in shards:
        if not own:
            lam_g.append(np.full((hq, ns), -np.inf))
            continue
        lam_g.append(row_lse(Qs_, Kp_[kept_token_index(own, n, c)], G))
    lam = lam_g[0]
    for g in range(1, W):
        lam = np.logaddexp(lam, lam_g[g])
    if norm == NORM_FULLROW:
        hkv = hq // G
        suf = np.stack([_logsumexp(_suffix_logits(Qs_, Ks, G, kvh), axis=-1) for kvh in range(hkv)])
        lam = np.logaddexp(lam, suf.reshape(hq, ns))
    cands = []
    A_full = np.zeros(m)
    for own in shards:
        if not own:
            continue
        # the shard's chunk scores: Eq. 1 over each owned chunk's own tokens
        a_g, _ = token_scores(Qs_, Kp_[kept_token_index(own, n, c)], G, lam=lam)
        A_g, pos = np.zeros(len(own)), 0
        for t, j in enumerate(own):
            lo, hi = chunk_range(j, n, c)
            A_g[t] = a_g[pos:pos + hi - lo].sum()
            pos += hi - lo
        A_full[own] = A_g
        loc = select_topk(A_g, min(k, len(own)))
        cands += [(A_g[t], own[int(t)]) for t in loc]
    top = sorted(cands, key=lambda t: (-t[0], t[1]))[:k]
    sel = np.array(sorted(j for _, j in top), dtype=np.int64)
    parts = []
    for g, own in enumerate(shards):
        mine = [j for j in sel if j in set(own)]
        parts.append(attention(Qs, Ks, Vs, Kp, Vp, kept_token_index(mine, n, c), G,
                               include_suffix=(g == W - 1)))
    O, lse = lse_merge(parts)
    return {"ids": sel, "out": O, "lse": lse, "A": A_full, "Lambda": lam}


def reprefill_periods(layers, c: int, k: int, G: int, period: int, norm: int = NORM_PREFIX):
    """Re-Prefill of consecutive layers with Periods (Def. 3):
    the chunk ids of layer l are identified at the first layer of its Period, p*floor(l/p), and
    reused by the other p-1 layers ("For the rest layers within the same Period, we reuse the same
    ContiguousChunk indices").  `layers` is a list of (Qs, Ks, Vs, Kp, Vp) per layer.
    Returns one reprefill_layer result per layer ('A' and 'gap' are those of the Period's first layer)."""
    if period < 1:
        raise ValueError("period must be >= 1")
    out = []
    first = None
    for l, (Qs, Ks, Vs, Kp, Vp) in enumerate(layers):
        if l % period == 0:
            first = reprefill_layer(Qs, Ks, Vs, Kp, Vp, c, k, G, norm=norm)
            out.append(first)
        else:
            r = reprefill_layer(Qs, Ks, Vs, Kp, Vp, c, k, G, norm=norm, sel=first["ids"])
            r["A"], r["gap"] = first["A"], first["gap"]
            out.append(r)
    return out

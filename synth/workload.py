"""Seeded synthetic Qwen2.5-shaped Re-Prefill workloads (recipe: DESIGN.md §3).

Counter-based generation: every tensor is drawn from its own numpy Philox
stream keyed on (seed, tensor id, layer, request), so any shard, rank or test
can regenerate exactly the same values independently.  Seed 42 is the paper's
(§5.1 "fixed random seed of 42").

Structure of the values (no method arithmetic here, only the recipe):

* Prefix keys carry N_TOPICS = 4 per-layer unit "topic" directions u_t per KV head.
  Chunk j of layer l has one salience field s_t[l, j] per topic (logit offsets on a
  geometric rank profile, see salience()) whose latent ranks follow an AR(1) process
  across layers (correlation ``rho``), so adjacent layers select overlapping chunk sets
  (the paper's cross-layer similarity).  Chunk 0 gets a sink boost
  and the last chunk a recency boost.
    Kp[i, h] = N(0, I) + sum_t s_t[j(i)] * u_t[h] * sqrt(d) / gamma
* A request's suffix queries point at a request-specific mixture of the topics, a unit
  weight vector w >= 0 (|N(0, I_4)| normalised), so different requests share part of
  their chunk sets (sink, recency, the topics they weigh alike -- something for the
  attention-guided cache to retain) and differ in the rest:
    Qs[r, h] = gamma * sum_t w_t u_t[h//G] + N(0, I)
  so the prefix logit q.k/sqrt(d) has mean ~ sum_t w_t s_t and O(1) noise: softmax
  rows are neither uniform nor one-hot.
* Prefix V, suffix K and suffix V are N(0, 1).

All values are rounded once to bf16 (round-to-nearest-even) for bf16 configs;
the oracle upcasts exactly those values.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 42

# tensor ids for the Philox key
_T_TOPIC, _T_KP, _T_VP, _T_QS, _T_KS, _T_VS, _T_MIX = range(2, 9)
_T_SAL = 16      # salience field t uses tensor id _T_SAL + t
N_TOPICS = 4


@dataclasses.dataclass(frozen=True)
class ShapeConfig:
    name: str
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    prefix_len: int
    chunk_size: int
    suffix_len: int
    budget_bp: int  # budget ratio in basis points
    dtype: str  # "bf16" or "fp32"

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def num_chunks(self) -> int:
        return -(-self.prefix_len // self.chunk_size)

    def replace(self, **kw) -> "ShapeConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs; Qwen2.5 head shapes.
CONFIGS = {
    "c1_0.5b": ShapeConfig("c1_0.5b", 1, 14, 2, 64, 2048, 16, 32, 1000, "fp32"),
    "c2_3b": ShapeConfig("c2_3b", 36, 16, 2, 128, 8192, 16, 64, 1000, "bf16"),
    "c3_7b": ShapeConfig("c3_7b", 28, 28, 4, 128, 32768, 16, 128, 1000, "bf16"),
    "c4_14b": ShapeConfig("c4_14b", 48, 40, 8, 128, 131072, 32, 256, 500, "bf16"),
    "c5_32b": ShapeConfig("c5_32b", 64, 40, 8, 128, 131072, 16, 256, 1000, "bf16"),
    # supplementary HBM-probe config: C3 shape with 8 suffix tokens
    "probe_7b_ns8": ShapeConfig("probe_7b_ns8", 28, 28, 4, 128, 32768, 16, 8, 1000, "bf16"),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    return (bf16_bits(x).astype(np.uint32) << 16).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) of float32 values, round-to-nearest-even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounded = u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return (rounded >> np.uint32(16)).astype(np.uint16)


def _rng(seed: int, tensor: int, layer: int, request: int = 0) -> np.random.Generator:
    key = (seed & 0xFFFFFFFF) | (tensor << 32) | (layer << 40) | (request << 64)
    return np.random.Generator(np.random.Philox(key=key))


def _finish(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    return bf16_round(x) if dtype == "bf16" else x


SPAN = 64.0   # logit range (nats) of the chunk-salience profile; see salience()
TOP = 2.0     # logit offset of the most salient ordinary chunk


def salience(cfg: ShapeConfig, layer: int, seed: int = SEED, rho: float = 0.9,
             span: float = SPAN, sink: float = 2.0, recency: float = 1.0):
    """N_TOPICS chunk-salience fields (logit offsets, nats) of length m for `layer`.

    Each field is a latent Gaussian z[l, j] following an AR(1) process across layers
    (correlation rho: adjacent layers select overlapping sets) mapped
    through its CDF onto a GEOMETRIC rank profile: s = TOP - span * (1 - Phi(z)), so the
    attention mass of chunk ranks decays exponentially (about span/m nats per rank; C3:
    0.031) and the top-10% of chunks holds most of a row's mass ("only a small set of important
    tokens ... is required").  The per-rank log-spacing is what keeps the k-th and (k+1)-th chunk
    scores apart (the Q11 gate of SURVEY §8(c): >= 95% of C3 draws strict);
    a Zipf profile rank^-1 would space them 1/k ~ 0.5% apart and fail the gate in ~1 draw
    of 5.  Chunk 0 gets a sink boost and the last chunk a recency boost above the top."""
    from scipy.special import ndtr  # standard normal CDF

    m = cfg.num_chunks
    out = []
    for t in range(_T_SAL, _T_SAL + N_TOPICS):
        z = _rng(seed, t, 0).standard_normal(m)
        for l in range(1, layer + 1):
            eps = _rng(seed, t, l).standard_normal(m)
            z = rho * z + math.sqrt(1.0 - rho * rho) * eps
        s = TOP - span * (1.0 - ndtr(z))
        s[0] = TOP + sink
        s[-1] = TOP + recency
        out.append(s)
    return out


def _topics(cfg: ShapeConfig, layer: int, seed: int):
    """[N_TOPICS, Hkv, d] unit topic directions of one layer."""
    g = _rng(seed, _T_TOPIC, layer)
    u = g.standard_normal((N_TOPICS, cfg.num_kv_heads, cfg.head_dim))
    u /= np.linalg.norm(u, axis=-1, keepdims=True)
    return u


def request_mix(request: int, seed: int = SEED) -> np.ndarray:
    """Unit topic weights w >= 0 of one request (|N(0, I)| normalised, uniform on the positive
    orthant of the sphere)."""
    w = np.abs(_rng(seed, _T_MIX, 0, request).standard_normal(N_TOPICS))
    return w / np.linalg.norm(w)


GAMMA = 4.0


def make_prefix(cfg: ShapeConfig, layer: int, seed: int = SEED, **sal_kw):
    """Prefix K, V of one layer, token-major [n, Hkv, d] (float32 holding bf16 values)."""
    n, hkv, d, c = cfg.prefix_len, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size
    sal = salience(cfg, layer, seed, **sal_kw)
    u = _topics(cfg, layer, seed)
    tok_chunk = np.arange(n) // c
    k = _rng(seed, _T_KP, layer).standard_normal((n, hkv, d), dtype=np.float32)
    scale = math.sqrt(d) / GAMMA
    for t in range(N_TOPICS):
        k += (sal[t][tok_chunk, None, None] * u[t][None]).astype(np.float32) * np.float32(scale)
    v = _rng(seed, _T_VP, layer).standard_normal((n, hkv, d), dtype=np.float32)
    return _finish(k, cfg.dtype), _finish(v, cfg.dtype)


def make_request(cfg: ShapeConfig, layer: int, request: int = 0, seed: int = SEED,
                 suffix_len: int | None = None):
    """Suffix Q [n_s, Hq, d], K, V [n_s, Hkv, d] of one request at one layer."""
    ns = cfg.suffix_len if suffix_len is None else suffix_len
    hq, hkv, d, G = cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.group
    w = request_mix(request, seed)
    dirn = np.tensordot(w, _topics(cfg, layer, seed), axes=1)  # [Hkv, d]
    q = _rng(seed, _T_QS, layer, request).standard_normal((ns, hq, d), dtype=np.float32)
    q += (GAMMA * dirn[np.arange(hq) // G][None]).astype(np.float32)
    ks = _rng(seed, _T_KS, layer, request).standard_normal((ns, hkv, d), dtype=np.float32)
    vs = _rng(seed, _T_VS, layer, request).standard_normal((ns, hkv, d), dtype=np.float32)
    return _finish(q, cfg.dtype), _finish(ks, cfg.dtype), _finish(vs, cfg.dtype)

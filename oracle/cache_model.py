"""Reference model of the attention-guided HBM chunk cache (TEST INFRASTRUCTURE).

Follows PAPER.md §4.4 (lines 424-455) step by step, specialised to the
B200 design of SURVEY §8(a) A4/A6/A9 (per-layer slot partitions):

* every (layer, chunk) keeps I (cumulative importance) and F (access count),
  including chunks not resident (the "in-memory table");
* S_j = I_j * F_j  (Eq. 2);
* before a load, the requested ids are checked against the cache;
  misses take free slots (ascending slot index), then slots of evicted residents:
  the lowest (S, j) residents that are not requested ("Both heaps will evict
  low-scored ContiguousChunks"; ties by (S, l, j));
* after the layer: I_j += A_j, F_j += 1 for the selected ids.

Ablation policies ("w/o AC: ContiguousKV using LFU as the cache
policy"): policy="lfu" ranks residents by S_j = F_j alone,
policy="lru" by the request index of the chunk's last selection (the `tick` passed to
update); the victim rule (lowest (S, j), never a requested chunk) is the same.

global_heap=True follows PAPER.md:447 ("a single global GPU heap") literally: one pool of
L * slots_per_layer slots serves every layer, and the victims of a plan are the lowest
(S, layer, chunk) residents of ANY layer that the plan does not request (SPEC.md:414 tie order).

Pure integer/slot bookkeeping plus the float compare of S; the GPU planner must
reproduce this exactly when S values are exact (integers), and the tests use such.
"""
from __future__ import annotations

import numpy as np


class CacheModel:
    POLICIES = ("attn", "lfu", "lru")

    def __init__(self, num_layers: int, num_chunks: int, slots_per_layer: int, policy: str = "attn",
                 global_heap: bool = False):
        assert policy in self.POLICIES, policy
        self.policy = policy
        self.L, self.m, self.P = num_layers, num_chunks, slots_per_layer
        self.global_heap = global_heap
        self.slot_of = np.full((num_layers, num_chunks), -1, dtype=np.int64)
        # pools: one per layer, or one shared pool; owner entries are (layer, chunk) or None
        npools, size = (1, num_layers * slots_per_layer) if global_heap else (num_layers, slots_per_layer)
        self.owner = [[None] * size for _ in range(npools)]
        self.I = np.zeros((num_layers, num_chunks))
        self.F = np.zeros((num_layers, num_chunks), dtype=np.int64)
        self.T = np.zeros((num_layers, num_chunks), dtype=np.int64)  # last-selection tick

    def _pool(self, layer: int):
        return self.owner[0] if self.global_heap else self.owner[layer]

    def score(self, layer: int) -> np.ndarray:
        """S_j = I_j x F_j  (Eq. 2); F_j (LFU) or the last-use tick (LRU) for the ablations."""
        if self.policy == "lfu":
            return self.F[layer].astype(np.float64)
        if self.policy == "lru":
            return self.T[layer].astype(np.float64)
        return self.I[layer] * self.F[layer]

    def plan(self, layer: int, ids, limit: int | None = None):
        """Hit/miss check and slot assignment for `ids` at `layer`.

        Returns (hits, loads, victims): loads is a list of (chunk, slot) in ascending chunk order
        (at most `limit` misses are loaded: the prefetch quota); victims are evicted entries as
        (layer, chunk) pairs in the global-heap mode and chunk ids otherwise."""
        ids = [int(j) for j in sorted(ids)]
        req = set(ids)
        pool = self._pool(layer)
        hits = [j for j in ids if self.slot_of[layer, j] >= 0]
        misses = [j for j in ids if self.slot_of[layer, j] < 0]
        if limit is not None:
            misses = misses[:limit]
        free = [s for s in range(len(pool)) if pool[s] is None]
        need = len(misses) - len(free)
        victims = []
        if need > 0:
            resident = [pool[s] for s in range(len(pool))
                        if pool[s] is not None and not (pool[s][0] == layer and pool[s][1] in req)]
            resident.sort(key=lambda e: (self.score(e[0])[e[1]], e[0], e[1]))
            if need > len(resident):
                raise RuntimeError("cache too small for the requested set")
            victims = resident[:need]
        slots = free[:len(misses)] + [int(self.slot_of[l, j]) for l, j in victims]
        for l, j in victims:
            pool[self.slot_of[l, j]] = None
            self.slot_of[l, j] = -1
        loads = []
        for j, s in zip(misses, slots):
            self.slot_of[layer, j] = s
            pool[s] = (layer, j)
            loads.append((j, s))
        return hits, loads, (victims if self.global_heap else [j for _, j in victims])

    def update(self, layer: int, ids, A, tick: int = 0) -> None:
        """I_j += A_j, F_j += 1 for every selected chunk; T_j = tick."""
        for j in ids:
            self.I[layer, int(j)] += float(A[int(j)])
            self.F[layer, int(j)] += 1
            self.T[layer, int(j)] = tick

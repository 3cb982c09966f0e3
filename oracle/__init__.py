"""fp64 CPU oracle of the ContiguousKV Re-Prefill hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2601_13631_b200``) never imports it and shares no code with it.

Every function follows PAPER.md (arxiv 2601.13631) in its own notation; where
the paper is silent or garbled the reading is SURVEY.md §8(c) Q1-Q16, listed in
DESIGN.md §2.  Parity pins: tests/test_oracle_*.py.  Parity unpinned: none
(every function below has at least one independent pin).
"""
from .ckv_oracle import (  # noqa: F401
    NORM_PREFIX,
    NORM_FULLROW,
    budget_chunks,
    chunk_count,
    chunk_range,
    prefix_logits,
    row_lse,
    token_scores,
    chunk_scores,
    select_topk,
    score_gap,
    parity_gate,
    valid_relaxed_set,
    GAP_GATE,
    FLOOR_REL,
    kept_token_index,
    attention,
    lse_merge,
    reprefill_layer,
    reprefill_periods,
    sharded_reprefill_layer,
    shard_chunks,
    coverage_ratio,
)
from .cache_model import CacheModel  # noqa: F401
from .granularity import block_cover, read_amplification  # noqa: F401

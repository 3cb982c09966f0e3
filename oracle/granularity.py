"""Granularity / read-amplification accounting (TEST INFRASTRUCTURE).

PAPER.md §3.1 (lines 209-221) and §4.2 (lines 316-328): a store organised in coarse blocks of
B tokens (64 in IMPRESS / AttentionStore) must read every block that holds at
least one needed token, so read amplification RA = tokens read / tokens needed
("11 tokens ... stored across 9 chunks, resulting in a read amplification of 52", PAPER.md:220-221;
"16 tokens within the chunk ... a read amplification ratio of 4").  When the
selection unit equals the storage unit (ContiguousChunks, c = B) every byte read is needed
and RA = 1 ("zero read amplification").

Selection units are the method's chunks of u tokens (u = 1 is token-level, H2O-style,
selection); unit j covers tokens [j*u, min((j+1)*u, n)) (Eq. 1 range, Q5/Q6).  A coarse block b
covers tokens [b*B, min((b+1)*B, n)); the padded tail of the last block is not counted as read
(SPEC.md:165).
"""
from __future__ import annotations


def block_cover(ids, unit_tokens: int, block_tokens: int, n: int) -> list[int]:
    """Ascending ids of the B-token blocks holding at least one token of the selected units."""
    if unit_tokens < 1 or block_tokens < 1 or n < 1:
        raise ValueError("unit_tokens, block_tokens and n must be >= 1")
    blocks = set()
    for j in ids:
        j = int(j)
        for t in range(j * unit_tokens, min((j + 1) * unit_tokens, n)):
            blocks.add(t // block_tokens)
    return sorted(blocks)


def read_amplification(ids, unit_tokens: int, block_tokens: int, n: int) -> tuple[int, int, float]:
    """(tokens_read, tokens_needed, RA) of loading the selected units from a B-token block store."""
    needed = sum(min((int(j) + 1) * unit_tokens, n) - int(j) * unit_tokens for j in set(int(x) for x in ids))
    read = sum(min((b + 1) * block_tokens, n) - b * block_tokens
               for b in block_cover(ids, unit_tokens, block_tokens, n))
    return read, needed, (read / needed if needed else 0.0)

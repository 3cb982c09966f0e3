"""NEXT-4 granularity study: read amplification and host-link bytes of token-level
(c = 1, H2O-style) selection served from a coarse 64-token block store (IMPRESS / AttentionStore,
PAPER.md:324) versus ContiguousChunk selection served from a store with the same granularity
(c = 16), on the real gather engine.

C3 shape (Qwen2.5-7B, 32K prefix, 28/4 heads, d = 128, bf16), layer 0, request r, 10% budget:
  aligned:  c = 16 selection (k = 204 chunks) -> RA from ckv_block_cover at B = 16 (= 1) and 64;
  token:    c = 1 selection (k = 3276 tokens) -> the 64-token blocks covering them (and 16-token);
  each covered set is then loaded cold (ckv_load_chunks after ckv_reset_cache) from a store of
  that granularity and timed with CUDA events: link bytes, us, GB/s.

    python scripts/ra_study.py [--out gpurun_out/ra_study.json] [--requests 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_13631_b200 import Context, ckv_budget_chunks  # noqa: E402
from synth import CONFIGS, make_prefix, make_request  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/ra_study.json")
    ap.add_argument("--requests", type=int, default=4)
    args = ap.parse_args()
    cfg = CONFIGS["c3_7b"]
    n, dev = cfg.prefix_len, torch.device("cuda", 0)
    kp, vp = make_prefix(cfg, 0)
    kp, vp = torch.from_numpy(kp).to(dev, torch.bfloat16), torch.from_numpy(vp).to(dev, torch.bfloat16)
    shape = (1, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim)

    def ctx_for(c, k, P):
        ctx = Context(*shape, c, n, cfg.suffix_len, dtype="bf16", budget_chunks=k, cache_slots=P)
        ctx.store_prefix(0, kp, vp)
        return ctx

    sel = {}
    for c in (16, 1):
        k = ckv_budget_chunks(n, c, cfg.budget_bp)
        sel[c] = ctx_for(c, k, k)
    stores = {B: ctx_for(B, -(-n // B), -(-n // B)) for B in (16, 64)}
    rec_bytes = {B: 2 * cfg.num_kv_heads * B * cfg.head_dim * 2 for B in (16, 64)}
    rows = []
    for r in range(args.requests):
        q, ks, vs = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in make_request(cfg, 0, r))
        for c, ctx in sel.items():
            out = torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device=dev)
            ids = torch.empty(ctx.k, dtype=torch.int32, device=dev)
            ctx.reset_cache()
            ctx.reprefill_layer(0, q, ks, vs, out=out, ids=ids)
            needed = ctx.k * c
            for B, store in stores.items():
                blocks, nb = ctx.block_cover(ids, B)
                nb = int(nb.item())
                store.reset_cache()
                store.reset_stats()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for b0 in range(0, nb, store.k):  # ckv_load_chunks takes at most k ids per call
                    store.load_chunks(0, blocks[b0:min(nb, b0 + store.k)])
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3
                st = store.get_stats()
                assert st["total_misses"] == nb and st["total_link_bytes_delta"] == nb * rec_bytes[B]
                read = min(nb * B, n)  # the last block of a 32K prefix is full
                row = {"request": r, "selection_unit": c, "store_block": B, "tokens_needed": needed,
                       "blocks_read": nb, "tokens_read": read, "RA": read / needed,
                       "link_MB": st["total_link_bytes_delta"] / 1e6, "gather_us": us,
                       "link_GBs": st["total_link_bytes_delta"] / us / 1e3,
                       "needed_GBs": needed * rec_bytes[B] / B / us / 1e3}
                rows.append(row)
                print(json.dumps(row), flush=True)
    for ctx in list(sel.values()) + list(stores.values()):
        ctx.close()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"workload": f"c3_7b layer 0, 10% budget, requests 0..{args.requests - 1}", "rows": rows},
                  f, indent=1)


if __name__ == "__main__":
    main()

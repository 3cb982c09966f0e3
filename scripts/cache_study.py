"""NEXT-2 cache study: attention-guided retention vs LFU vs LRU, with and without
speculative prefetch -- the ablation of PAPER.md:605-623 ("w/o AC": LFU as the cache policy;
"w/o P": no prefetching) on a synthetic multi-request shared-prefix workload.

Workload: the C3 shape (Qwen2.5-7B, 28 layers, 32K prefix, c = 16, n_s = 128, bf16); R = 16
distinct requests (each its own topic mixture, synth.make_request) drawn 48 times with Zipf(1)
popularity (seed 42); the first 16 draws warm the cache ("warm up one full pass"),
the other 32 are measured.  Budgets 10% and 25% (the ablation's ratio); per-layer
HBM cache of P = 1.25k, 1.5k, 2k, 3k slots (the prefetch quota, min(k, P - k), is part of P when
prefetch is on, so both variants have the same HBM).  Per variant:
hit rate, host-link MB per layer (critical-path delta and speculative), and the median eager
us/layer over the measured requests (CUDA events on the launching stream).

    python scripts/cache_study.py [--out gpurun_out/cache_study.json] [--draws 48]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_13631_b200 import CKV_FLAG_GLOBAL_HEAP, Context, ckv_budget_chunks  # noqa: E402
from synth import CONFIGS, make_prefix, make_request  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cache_study.json")
    ap.add_argument("--draws", type=int, default=48)
    ap.add_argument("--requests", type=int, default=16)
    ap.add_argument("--budgets", default="1000,2500")
    ap.add_argument("--config", default="c3_7b", help="synth config (c5_32b: the shared-prefix C5 shape)")
    ap.add_argument("--layers", type=int, default=0, help="run only the first L layers (per-layer cache "
                    "partitions make layers independent; 0 = all)")
    ap.add_argument("--slots", default="1.25,1.5,2,3", help="HBM slots per layer as multiples of k")
    ap.add_argument("--heaps", default="layer", help="comma list of 'layer' (per-layer pools) and 'global' "
                    "(one pool of L x slots shared by every layer, PAPER.md:447)")
    args = ap.parse_args()
    base = CONFIGS[args.config]
    if args.layers:
        base = base.replace(num_layers=args.layers)
    L, dev = base.num_layers, torch.device("cuda", 0)
    prefix = []
    for l in range(L):
        kp, vp = make_prefix(base, l)
        prefix.append((torch.from_numpy(kp).to(dev, torch.bfloat16), torch.from_numpy(vp).to(dev, torch.bfloat16)))
    R = args.requests
    reqs = [[[torch.from_numpy(x).to(dev, torch.bfloat16) for x in make_request(base, l, r)] for l in range(L)]
            for r in range(R)]
    g = np.random.default_rng(42)
    pop = 1.0 / np.arange(1, R + 1)
    draws = g.choice(R, size=args.draws, p=pop / pop.sum()).tolist()
    warm = min(R, args.draws // 3)
    outs = [torch.empty(base.suffix_len, base.num_q_heads, base.head_dim, dtype=torch.bfloat16, device=dev)
            for _ in range(L)]
    results = []
    for bp in [int(b) for b in args.budgets.split(",")]:
        k = ckv_budget_chunks(base.prefix_len, base.chunk_size, bp)
        ids = [torch.empty(k, dtype=torch.int32, device=dev) for _ in range(L)]
        mults = [float(x) for x in args.slots.split(",")]
        for heap, P, prefetch in [(h, int(k * f), pf) for h in args.heaps.split(",") for f in mults
                                  for pf in (True, False)]:
            quota = min(k, P - k) if prefetch else 0
            ctx = Context(L, base.num_q_heads, base.num_kv_heads, base.head_dim, base.chunk_size, base.prefix_len,
                          base.suffix_len, dtype="bf16", budget_bp=bp, prefetch_chunks=quota, cache_slots=P,
                          flags=CKV_FLAG_GLOBAL_HEAP if heap == "global" else 0)
            for l in range(L):
                ctx.store_prefix(l, *prefix[l])
            for policy in ("attn", "lfu", "lru"):
                ctx.set_cache_policy(policy)
                us = []
                for i, r in enumerate(draws):
                    if i == warm:
                        torch.cuda.synchronize()
                        ctx.reset_stats()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for l in range(L):
                        ctx.reprefill_layer(l, *reqs[r][l], out=outs[l], ids=ids[l])
                    e1.record()
                    torch.cuda.synchronize()
                    if i >= warm:
                        us.append(e0.elapsed_time(e1) * 1e3 / L)
                st = ctx.get_stats()
                nl = max(st["total_layers"], 1)
                sel = st["total_hits"] + st["total_misses"]
                row = {"budget_bp": bp, "k": k, "heap": heap, "slots_per_layer": P, "prefetch_quota": quota, "policy": policy,
                       "hit_rate": st["total_hits"] / max(sel, 1),
                       "delta_MB_per_layer": st["total_link_bytes_delta"] / nl / 1e6,
                       "spec_MB_per_layer": st["total_link_bytes_spec"] / nl / 1e6,
                       "spec_used_frac": st["total_spec_used"] / max(st["total_spec_loads"], 1),
                       "us_per_layer_median": statistics.median(us), "us_per_layer_mean": statistics.mean(us)}
                results.append(row)
                print(json.dumps(row), flush=True)
            ctx.close()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"workload": f"{args.config} shape ({L} layers), R={R} requests, {args.draws} Zipf(1) draws "
                               f"(first {warm} warm-up), seed 42", "draws": draws, "rows": results}, f, indent=1)


if __name__ == "__main__":
    main()

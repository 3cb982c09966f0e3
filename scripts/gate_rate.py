#!/usr/bin/env python
"""Q11 parity-gate pass rate of the synthetic workload (oracle only, CPU).

    python scripts/gate_rate.py [--cfg c3_7b] [--layers 0-9] [--requests 0-7] [--out f.json]

For each (layer, request) draw: the fp64 oracle's chunk scores A (Eq. 1), the k/k+1 gap
 and whether the strict (bit-exact ids) gate applies; also the row entropy
of the prefix softmax and the adjacent-layer top-k coverage.  Writes the
per-draw table and the pass fraction (DESIGN.md §4 quotes it)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from synth import CONFIGS, make_prefix, make_request  # noqa: E402


def rng(s):
    a, b = s.split("-") if "-" in s else (s, s)
    return list(range(int(a), int(b) + 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3_7b")
    ap.add_argument("--layers", default="0-9")
    ap.add_argument("--requests", default="0")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.cfg]
    k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    rows, prev = [], {}
    t0 = time.time()
    for l in rng(a.layers):
        kp, _ = make_prefix(cfg, l)
        for r in rng(a.requests):
            qs, ks, _ = make_request(cfg, l, r)
            ai, lam = O.token_scores(qs, kp, cfg.group)
            A = O.chunk_scores(ai, cfg.chunk_size)
            ids = O.select_topk(A, k)
            row = {"layer": l, "request": r, "gap": O.score_gap(A, k), "strict": bool(O.parity_gate(A, k)),
                   "top1_share": float(A.max() / A.sum()), "topk_share": float(A[ids].sum() / A.sum())}
            if (l - 1, r) in prev:
                row["coverage_prev"] = O.coverage_ratio(ids, prev[(l - 1, r)])
            prev[(l, r)] = ids
            rows.append(row)
            print(json.dumps(row), flush=True)
    rate = sum(r["strict"] for r in rows) / len(rows)
    # per layer: size of the union of the requests' selected sets (what an HBM cache must hold to
    # serve every request of the stream without host loads)
    unions = {}
    for (l, r), ids in prev.items():
        unions.setdefault(l, set()).update(int(x) for x in ids)
    cov = [r["coverage_prev"] for r in rows if "coverage_prev" in r]
    summ = {"cfg": a.cfg, "k": k, "draws": len(rows), "gate_pass_rate": rate,
            "coverage_prev_mean": float(np.mean(cov)) if cov else None,
            "topk_share_mean": float(np.mean([r["topk_share"] for r in rows])),
            "union_per_layer_mean": float(np.mean([len(u) for u in unions.values()])), "seconds": time.time() - t0}
    print(json.dumps(summ))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summ, "draws": rows}, f, indent=1)


if __name__ == "__main__":
    main()

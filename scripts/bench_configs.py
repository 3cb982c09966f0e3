#!/usr/bin/env python
"""Per-layer Re-Prefill timings on the other BASELINE.json configs (C1, C2 at its 36 layers, C4 at
its 128K prefix on one GPU, the C5 chunk-size x budget sweep) and the C3 headline shape, one JSON
record per configuration -> --out (default gpurun_out/bench_configs.json).

Per config: one request's layers replayed from a CUDA graph with every selected chunk resident
(warm, `us_per_layer`), the same from an empty HBM cache (`cold_us_per_layer`), the A1 score
kernel's average launch (library events) with its MUFU-roofline fraction, and the effective KV
GB/s of bench.py's metric.  C4/C5 run L_run layers of their shape (per-layer numbers do not
depend on L; the pinned host store of all 48 / 64 layers would be 24 / 32 GiB)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_13631_b200 as ckv  # noqa: E402
from synth import CONFIGS, make_prefix, make_request  # noqa: E402


def bytes_per_layer(cfg, k):
    e = 2 if cfg.dtype == "bf16" else 4
    return (cfg.prefix_len * cfg.num_kv_heads * cfg.head_dim * e + k * 2 * cfg.num_kv_heads * cfg.chunk_size *
            cfg.head_dim * e + 2 * cfg.suffix_len * cfg.num_kv_heads * cfg.head_dim * e)


def run(cfg, L, steps=5):
    dev = torch.device("cuda", 0)
    k = ckv.ckv_budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    ctx = ckv.Context(L, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len,
                      cfg.suffix_len, dtype=cfg.dtype, budget_bp=cfg.budget_bp, prefetch_chunks=k,
                      cache_slots=2 * k + k // 2)
    dt = ctx.torch_dtype
    for l in range(L):
        kp, vp = make_prefix(cfg, l)
        ctx.store_prefix(l, torch.from_numpy(kp).to(dev, dt), torch.from_numpy(vp).to(dev, dt))
    req = [[torch.from_numpy(x).to(dev, dt) for x in make_request(cfg, l, 0)] for l in range(L)]
    outs = [torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=dt, device=dev) for _ in range(L)]
    ids = [torch.empty(k, dtype=torch.int32, device=dev) for _ in range(L)]

    def step():
        for l in range(L):
            ctx.reprefill_layer(l, *req[l], out=outs[l], ids=ids[l])

    for _ in range(3):
        step()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(2):
        g.replay()

    def timed(fn, K):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    ms = timed(g.replay, steps)
    cold = []
    for _ in range(3):
        ctx.reset_cache()
        cold.append(timed(g.replay, 1))
    ctx.profile(True)
    for _ in range(2):
        step()
    pr = ctx.profile_read()
    ctx.profile(False)
    score_ms = pr["score"][0] / max(pr["score"][1], 1)
    exps = cfg.num_q_heads * cfg.suffix_len * cfg.prefix_len
    mufu_peak = 16 * 148 * 1.965e9
    bpl = bytes_per_layer(cfg, k)
    rec = {"config": cfg.name, "layers_run": L, "prefix": cfg.prefix_len, "chunk": cfg.chunk_size,
           "suffix": cfg.suffix_len, "heads": f"{cfg.num_q_heads}/{cfg.num_kv_heads}", "budget_bp": cfg.budget_bp,
           "k": k, "dtype": cfg.dtype, "us_per_layer": ms * 1e3 / L, "gbs": bpl / (ms * 1e-3 / L) / 1e9,
           "cold_us_per_layer": min(cold) * 1e3 / L, "score_kernel": ["simt", "tcgen05"][ctx.score_kernel_kind],
           "score_us": score_ms * 1e3, "score_mufu_frac_at_max_clock": exps / (score_ms * 1e-3) / mufu_peak,
           "stage_us_per_layer": {n: v[0] * 1e3 / max(v[1], 1) for n, v in pr.items() if v[1]}}
    ctx.close()
    del g
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/bench_configs.json")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    jobs = [("c1", CONFIGS["c1_0.5b"], 1), ("c2", CONFIGS["c2_3b"], 36), ("c3", CONFIGS["c3_7b"], 28),
            ("c4", CONFIGS["c4_14b"], 4)]
    for c in (4, 16, 64):
        for bp in (200, 500, 1000, 2500, 5000):
            cfg = CONFIGS["c5_32b"].replace(chunk_size=c, budget_bp=bp, name=f"c5_32b_c{c}_b{bp}")
            jobs.append((f"c5_c{c}_b{bp}", cfg, 2))
    out = []
    for tag, cfg, L in jobs:
        if a.only and not tag.startswith(a.only):
            continue
        t = time.time()
        try:
            r = run(cfg, L)
        except Exception as ex:  # report and go on (e.g. a shape outside the compiled kernels)
            r = {"config": cfg.name, "error": str(ex)[:300]}
        r["wall_s"] = time.time() - t
        print(json.dumps(r), flush=True)
        out.append(r)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

"""Host-link efficiency of the zero-copy chunk gather (A5) vs a pinned cudaMemcpy of the same bytes.

C3 records (32 KiB, 7B shape), one layer store; ckv_load_chunks demand-loads n ascending random
chunk ids into an empty HBM cache (the gather engine of A5/A6), CUDA events around it; the
reference is torch's pinned H2D copy of n * 32 KiB.  Prints one JSON line per n.
    python scripts/link_probe.py [n ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_13631_b200 import Context
from synth import CONFIGS, make_prefix
cfg = CONFIGS["c3_7b"]
m = cfg.num_chunks
dev = torch.device("cuda", 0)
kp, vp = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in make_prefix(cfg, 0))
ctx = Context(1, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len, cfg.suffix_len,
              dtype="bf16", budget_chunks=m, cache_slots=m)
ctx.store_prefix(0, kp, vp)
rec = 2 * cfg.num_kv_heads * cfg.chunk_size * cfg.head_dim * 2
g = np.random.default_rng(0)
for n in [int(x) for x in sys.argv[1:]] or [64, 204, 512, 1024, 2048]:
    ids = torch.from_numpy(np.sort(g.choice(m, n, replace=False)).astype(np.int32)).to(dev)
    ts = []
    for rep in range(5):
        ctx.reset_cache()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.load_chunks(0, ids)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = torch.empty(n * rec, dtype=torch.uint8).pin_memory()
    d = torch.empty(n * rec, dtype=torch.uint8, device=dev)
    tm = []
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        tm.append(e0.elapsed_time(e1))
    b = n * rec
    print(json.dumps({"chunks": n, "bytes": b, "gather_us": min(ts) * 1e3, "gather_gbs": b / min(ts) / 1e6,
                      "memcpy_us": min(tm) * 1e3, "memcpy_gbs": b / min(tm) / 1e6}), flush=True)

"""Debug: kernel-end timeline of one graph-replayed C3 step (CKV_TIMELINE=1, printed at close)."""
import os, sys
os.environ.setdefault("CKV_LIBRARY", "tuning")  # env knobs exist only in the tuning build
os.environ["CKV_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O
from paper_2601_13631_b200 import Context
from synth import CONFIGS, make_prefix, make_request
cfg = CONFIGS["c3_7b"]
k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
ctx = Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len,
              cfg.suffix_len, dtype="bf16", budget_bp=cfg.budget_bp, prefetch_chunks=k, cache_slots=k + k + k // 2)
for l in range(cfg.num_layers):
    kp, vp = make_prefix(cfg, l)
    ctx.store_prefix(l, torch.from_numpy(kp).cuda().bfloat16(), torch.from_numpy(vp).cuda().bfloat16())
R = 16
reqs = [[[torch.from_numpy(x).cuda().bfloat16() for x in make_request(cfg, l, r)] for l in range(cfg.num_layers)]
        for r in range(R)]
from bench import request_sequence
seq = request_sequence(64) if os.environ.get("TL_REQ", "steady") == "steady" else [0] * 64
outs = [torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
        for _ in range(cfg.num_layers)]
ids = [torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(cfg.num_layers)]
def step(r):
    for l in range(cfg.num_layers):
        ctx.reprefill_layer(l, *reqs[r][l], out=outs[l], ids=ids[l])
for i in range(24):
    step(seq[i])
mode = os.environ.get("TL_MODE", "eager")
if mode == "graph":
    gs = []
    for r in range(R):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(r)
        gs.append(g)
    for i in range(24, 32):
        gs[seq[i]].replay()
else:
    for i in range(24, 32):
        step(seq[i])
torch.cuda.synchronize()
ctx.close()

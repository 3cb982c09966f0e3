"""Profiling driver: a few C3 layers through the C-ABI (product library), for ncu captures.
    ncu ... python scripts/prof_layer.py [layers] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import CONFIGS, make_request
from tests.gpu_util import make_ctx, to_dev
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS["c3_7b"].replace(num_layers=L)
ctx, _ = make_ctx(cfg, prefetch=204, cache_slots=510)
reqs = [[to_dev(x, torch.bfloat16) for x in make_request(cfg, l, 0)] for l in range(L)]
for _ in range(reps):
    for l in range(L):
        ctx.reprefill_layer(l, *reqs[l])
torch.cuda.synchronize()
print("done")

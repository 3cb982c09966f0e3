"""A/B timing of the tcgen05 score kernel variants (CKV_SCORE_POLY = pairs of every 8 exp2 pairs on the FMA pipe)."""
import os, sys, json
os.environ.setdefault("CKV_LIBRARY", "tuning")  # env knobs exist only in the tuning build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from synth import CONFIGS, make_request
from tests.gpu_util import make_ctx, to_dev
cfg = CONFIGS["c3_7b"].replace(num_layers=4)
ctx, prefix = make_ctx(cfg)
reqs = [[to_dev(x, torch.bfloat16) for x in make_request(cfg, l, 0)] for l in range(cfg.num_layers)]
A = torch.empty(ctx.m_local, device="cuda")
for rep in range(2):
    for l in range(cfg.num_layers):
        ctx.reprefill_layer(l, *reqs[l], chunk_scores=A if l == 0 else None)
torch.cuda.synchronize()
ref = O.reprefill_layer(*make_request(cfg, 0, 0), *prefix[0], cfg.chunk_size, ctx.k, cfg.group)
Ad = A.cpu().numpy().astype(np.float64)
ctx.profile(True)
for rep in range(5):
    for l in range(cfg.num_layers):
        ctx.reprefill_layer(l, *reqs[l])
pr = ctx.profile_read()
print(json.dumps({"poly": os.environ.get("CKV_SCORE_POLY", "default"), "score_us": pr["score"][0] / pr["score"][1] * 1e3,
                  "A_rel_max": float((np.abs(Ad - ref["A"]) / np.maximum(ref["A"], 1e-30 * ref["A"].sum())).max()),
                  "ids_equal": bool(np.array_equal(np.sort(np.argsort(-Ad, kind="stable")[:ctx.k]), ref["ids"]))}))

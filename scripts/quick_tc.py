"""Quick tcgen05 score-kernel sanity check (one small bf16 layer) for GPU bring-up."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from synth import CONFIGS
from tests.gpu_util import make_ctx, run_layers, check_layer
cfg = CONFIGS["c3_7b"].replace(num_layers=1, prefix_len=4096, suffix_len=32)
k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
ctx, prefix = make_ctx(cfg)
print("score kernel kind", ctx.score_kernel_kind, "attn kind", ctx.attn_kernel_kind, flush=True)
t = time.time()
r = run_layers(ctx, cfg, prefix, [0])[0]
print("ran in", time.time() - t, flush=True)
ref = O.reprefill_layer(r["qs"], r["ks"], r["vs"], *prefix[0], cfg.chunk_size, k, cfg.group)
rel = np.abs(r["A"] - ref["A"]) / ref["A"]
print("A rel max", rel.max(), "A sum", r["A"].sum(), ref["A"].sum(), flush=True)
print(check_layer(r["ids"], r["out"], r["A"], r["qs"], r["ks"], r["vs"], *prefix[0], cfg, k))

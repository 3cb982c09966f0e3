"""Debug: per-event timeline of CTA 0 of the tcgen05 attention kernel (CKV_ATTN_TRACE=1)."""
import os, sys
os.environ.setdefault("CKV_LIBRARY", "tuning")  # env knobs exist only in the tuning build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CKV_ATTN_TRACE"] = "1"
import torch
from synth import CONFIGS
from tests.gpu_util import make_ctx, run_layers
cfg = CONFIGS["c3_7b"].replace(num_layers=2)
ctx, prefix = make_ctx(cfg, prefetch=204)
for rep in range(3):
    run_layers(ctx, cfg, prefix, [0, 1], request=rep, with_A=False)
    print("---", flush=True)

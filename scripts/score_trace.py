"""Debug: per-event timeline of CTA 0 of the tcgen05 score kernel (CKV_SCORE_TRACE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CKV_SCORE_TRACE"] = "1"
import torch
from synth import CONFIGS
from tests.gpu_util import make_ctx, run_layers
cfg = CONFIGS["c3_7b"].replace(num_layers=1)
ctx, prefix = make_ctx(cfg)
for rep in range(3):
    run_layers(ctx, cfg, prefix, [0], request=rep, with_A=False)
    print("---", flush=True)

"""Debug: per-unit event timeline of CTA 0 of the tcgen05 score kernel (tuning build,
CKV_SCORE_TRACE=1): Q landed, accumulator free (MMAs issued), MMA done, accumulator released,
epilogue done -- microseconds since the first event."""
import os, sys
os.environ.setdefault("CKV_LIBRARY", "tuning")  # env knobs exist only in the tuning build
os.environ["CKV_SCORE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import CONFIGS, make_request
from tests.gpu_util import make_ctx, to_dev
cfg = CONFIGS[os.environ.get("TRACE_CFG", "c3_7b")].replace(num_layers=1)
ctx, _ = make_ctx(cfg)
q, k_, v_ = (to_dev(x, torch.bfloat16) for x in make_request(cfg, 0, 0))
for rep in range(3):
    ctx.reprefill_layer(0, q, k_, v_)
    torch.cuda.synchronize()
    print("---", flush=True)

"""Debug: test_c1_fp32_full_config followed by the token-level c=1 fp32 case; per-row errors."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gc
import oracle as O
import tests.test_gpu_parity as t
from tests.gpu_util import make_ctx, run_layers
from synth import ShapeConfig
if os.environ.get("FIRST", "1") == "1":
    t.test_c1_fp32_full_config()
if os.environ.get("GC", "0") == "1":
    gc.collect(); torch.cuda.synchronize()
cfg = ShapeConfig("tok", 1, 4, 2, 64, 700, 1, 5, 1000, "fp32")
ctx, prefix = make_ctx(cfg, k=37)
res = run_layers(ctx, cfg, prefix, [0])[0]
ref = O.reprefill_layer(res["qs"], res["ks"], res["vs"], *prefix[0], cfg.chunk_size, 37, cfg.group)
out = res["out"].astype(np.float64)
err = np.abs(out - ref["out"]).max(-1) / np.abs(ref["out"]).max(-1)
print("ids equal", res["ids"].tolist() == ref["ids"].tolist())
print("row err (r x h):\n", np.array2string(err, precision=2))
print("gpu out[0,0,:4]", out[0, 0, :4], "ref", ref["out"][0, 0, :4])

"""Small workloads for compute-sanitizer (scripts/sanitize.sh): C1 (fp32 SIMT path), a ragged bf16
tcgen05 case with prefetch and periods, the global heap, the V-only store, and two logical ranks
of the fused sharded exchange."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_13631_b200 import CKV_FLAG_GLOBAL_HEAP, CKV_FLAG_V_ONLY_STORE
from synth import ShapeConfig, CONFIGS, make_request
from tests.gpu_util import make_ctx, run_layers, to_dev
small = ShapeConfig("s", 2, 8, 2, 128, 3001, 16, 40, 1000, "bf16")
for cfg, kw in ((CONFIGS["c1_0.5b"], {}), (small, dict(prefetch=8, k=16)),
                (small, dict(k=16, flags=CKV_FLAG_GLOBAL_HEAP, cache_slots=24)),
                (small, dict(k=16, prefetch=8, flags=CKV_FLAG_V_ONLY_STORE))):
    ctx, prefix = make_ctx(cfg, **kw)
    run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=1)
    if "flags" not in kw and cfg.dtype == "bf16":
        ctx.set_period(2, 2)
        run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=2)
    ctx.close()
# two logical ranks, fused exchange
W = 2
ctxs = [make_ctx(small, shard=g, W=W, k=16)[0] for g in range(W)]
for c in ctxs:
    c.exchange_attach(ctxs)
streams = [torch.cuda.Stream() for _ in range(W)]
for l in range(small.num_layers):
    q, k_, v_ = (to_dev(x, torch.bfloat16) for x in make_request(small, l, 0))
    torch.cuda.synchronize()
    for g, c in enumerate(ctxs):
        with torch.cuda.stream(streams[g]):
            c.reprefill_layer(l, q, k_, v_, stream=streams[g])
    torch.cuda.synchronize()
for c in ctxs:
    c.close()
print("sanitize case done")

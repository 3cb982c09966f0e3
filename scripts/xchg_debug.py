"""Debug: progress of the fused exchange with W logical ranks on one GPU (per-call host timing,
stream completion and the exchange counters of every rank, polled for a few seconds)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import ShapeConfig, make_request
from tests.gpu_util import make_ctx, to_dev
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = ShapeConfig("dbg", 1, 28, 4, 128, 4000, 16, 40, 1000, "bf16")
ctxs = [make_ctx(cfg, shard=g, W=W)[0] for g in range(W)]
for c in ctxs:
    c.exchange_attach(ctxs)
streams = [torch.cuda.Stream() for _ in range(W)]
qs, ks, vs = make_request(cfg, 0, 0)
q, k_, v_ = (to_dev(x, torch.bfloat16) for x in (qs, ks, vs))
torch.cuda.synchronize()
print("flags before", [c.test_exchange_flags() for c in ctxs], flush=True)
for g, c in enumerate(ctxs):
    t = time.time()
    with torch.cuda.stream(streams[g]):
        c.reprefill_layer(0, q, k_, v_, stream=streams[g])
    print(f"rank {g} enqueued in {time.time() - t:.3f}s", flush=True)
for i in range(20):
    print(i, "done", [s.query() for s in streams], "flags", [c.test_exchange_flags() for c in ctxs], flush=True)
    if all(s.query() for s in streams):
        break
    time.sleep(0.5)
print("finished", all(s.query() for s in streams), flush=True)
os._exit(0)

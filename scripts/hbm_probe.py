"""SURVEY §8(d) HBM probe: the C3 prefix with an 8-token suffix (56 GQA rows per KV head), where A1
streams the 33.5 MB of probe keys per layer below both compute ridges.  Run under ncu for the
kernel's own duration and DRAM bytes:
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:score_tc python scripts/hbm_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_13631_b200 import Context, ckv_budget_chunks  # noqa: E402
from synth import CONFIGS, make_prefix, make_request  # noqa: E402

cfg = CONFIGS["probe_7b_ns8"].replace(num_layers=4)
k = ckv_budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
ctx = Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len,
              cfg.suffix_len, dtype="bf16", budget_bp=cfg.budget_bp)
for l in range(cfg.num_layers):
    kp, vp = make_prefix(cfg, l)
    ctx.store_prefix(l, torch.from_numpy(kp).cuda().bfloat16(), torch.from_numpy(vp).cuda().bfloat16())
reqs = [[torch.from_numpy(x).cuda().bfloat16() for x in make_request(cfg, l)] for l in range(cfg.num_layers)]
for rep in range(3):
    for l in range(cfg.num_layers):
        ctx.reprefill_layer(l, *reqs[l])
torch.cuda.synchronize()
print("ok")

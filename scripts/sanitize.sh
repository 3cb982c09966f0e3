#!/bin/bash
# compute-sanitizer memcheck / racecheck on small configurations (GPU box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/san_case.py << 'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from synth import ShapeConfig, CONFIGS
from tests.gpu_util import make_ctx, run_layers
for cfg in (CONFIGS["c1_0.5b"], ShapeConfig("s", 2, 8, 2, 128, 3001, 16, 40, 1000, "bf16")):
    ctx, prefix = make_ctx(cfg, prefetch=8, k=16 if cfg.dtype == "bf16" else 0)
    run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=1)
    ctx.close()
print("sanitize case done")
PY
timeout 900 compute-sanitizer --tool memcheck --leak-check no python /tmp/san_case.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
tail -5 gpurun_out/memcheck.log

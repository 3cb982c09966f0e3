#!/bin/bash
# Score-kernel exp2 split sweep on the tuning build: bench-event time and accuracy per variant.
#   bash scripts/score_sweep.sh 0 2 3 4 5 6   -> gpurun_out/score_sweep.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2601_13631_b200.build --tuning > /dev/null
for P in "$@"; do
  CKV_LIBRARY=tuning CKV_SCORE_POLY=$P timeout 300 python scripts/score_ab.py 2>&1 | tail -1 | tee -a gpurun_out/score_sweep.log
done

#!/bin/bash
# Score-kernel timing variants (tuning build): CKV_SCORE_DBG 0 full, 1 no epilogue math, 3 math without
# stores; per-unit trace of CTA 0.
cd "$(dirname "$0")/.."
for D in ${DBGS:-0 1 3}; do
  echo "== CKV_SCORE_DBG=$D"
  CKV_SCORE_DBG=$D timeout 120 python scripts/score_trace.py 2>&1 | tail -11
done

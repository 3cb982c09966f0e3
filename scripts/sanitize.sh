#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small configurations (GPU box) ->
# gpurun_out/{memcheck,racecheck,synccheck}.log  (scripts/san_case.py)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
for T in memcheck racecheck synccheck; do
  extra=""
  [ "$T" == "memcheck" ] && extra="--leak-check no"
  timeout 1200 compute-sanitizer --tool $T $extra python scripts/san_case.py > gpurun_out/$T.log 2>&1
  echo "$T rc=$?" >> gpurun_out/$T.log
  tail -3 gpurun_out/$T.log
done

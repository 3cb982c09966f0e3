#!/bin/bash
# One GPU round: quick tcgen05 check, GPU tests, smoke, bench; optional ncu launch list + full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python scripts/quick_tc.py > gpurun_out/quick.log 2>&1 || { echo "quick failed"; tail -20 gpurun_out/quick.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
if [ "$1" == "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1300 -c 400 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_launch.log 2>&1
  for K in score_tc attn_tc compact_kv row_lse chunk_sum topk_plan2 attn_combine; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 1 \
       -o gpurun_out/$K python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_$K.log 2>&1
  done
fi
[ "$1" == "ncu" ] && python scripts/ncu_summary.py gpurun_out/ncu_summary.md gpurun_out/launches.csv \
  gpurun_out/score_tc.ncu-rep gpurun_out/attn_tc.ncu-rep gpurun_out/compact_kv.ncu-rep gpurun_out/row_lse.ncu-rep \
  gpurun_out/chunk_sum.ncu-rep gpurun_out/topk_plan2.ncu-rep gpurun_out/attn_combine.ncu-rep > /dev/null 2>&1
tail -n 3 gpurun_out/quick.log gpurun_out/pytest_gpu.log gpurun_out/smoke.log
tail -c 600 gpurun_out/bench.log

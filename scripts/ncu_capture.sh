#!/bin/bash
# ncu launch list of one bench step + one full capture per hot kernel, summarised to gpurun_out/ncu_summary.md
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1300 -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_launch.log 2>&1
K_LIST=${K_LIST:-"score_tc attn_tc compact_kv row_lse chunk_sum topk_plan2 attn_combine"}
REPS=""
for K in $K_LIST; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 1 \
     -o gpurun_out/$K python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_$K.log 2>&1
  REPS="$REPS gpurun_out/$K.ncu-rep"
done
python scripts/ncu_summary.py gpurun_out/ncu_summary.md gpurun_out/launches.csv $REPS > /dev/null 2>&1
python scripts/ktimes.py gpurun_out/launches.csv | head -16

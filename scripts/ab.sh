#!/bin/bash
# A/B of source variants (build.py --variant NAME -> libckv_NAME.so): warm graph-step time of the
# bench (twice each, interleaved) and, with KT=1, the ncu per-kernel launch list of prof_layer.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for V in $VARIANTS; do
    echo "== $V rep $rep: $(CKV_LIBRARY=variant:$V timeout 300 python bench.py --quick 2>&1 | tail -1)"
  done
done
if [ "$KT" == "1" ]; then
  for V in $VARIANTS; do
    CKV_LIBRARY=variant:$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/l_$V.csv python scripts/prof_layer.py 2 3 > /dev/null 2>&1
    echo "== kernels $V"; python scripts/ktimes.py gpurun_out/l_$V.csv | grep -v pack_ | head -12
  done
fi

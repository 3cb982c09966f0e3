# Tuning sweep of the score kernel variants (CKV_SCORE_POLY values given as arguments):
# one ncu launch list per variant -> gpurun_out/np_<P>.csv (summarise with scripts/np_summary.py)
mkdir -p gpurun_out
for P in "$@"; do
  CKV_LIBRARY=tuning CKV_SCORE_POLY=$P timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:score_tc --csv python scripts/score_ab.py > gpurun_out/np_$P.csv 2>&1
done

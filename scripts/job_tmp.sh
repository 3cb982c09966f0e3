cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for i in 1 2; do echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 1300 -c 400 --csv \
     --log-file gpurun_out/launches_warm.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_launch_warm.log 2>&1
python scripts/ktimes.py gpurun_out/launches_warm.csv 2>&1 | head -30

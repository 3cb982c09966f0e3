cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "topk or c3 or c2" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__cycles_active.max --clock-control none --cache-control none -k regex:topk -s 20 -c 3 python bench.py --steps 1 --warmup 3 --no-cpu --no-graph 2>&1 | grep -E "duration|cycles_active" | head -6

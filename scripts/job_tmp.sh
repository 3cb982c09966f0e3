cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
grep -B2 -A30 "Error\|FAIL" gpurun_out/pytest_gpu.log | head -50
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_v.log').read().strip().splitlines()[-1]); print(d['us_per_layer'], d['cold_cache'], d['cold_cache_v_only'])"
tail -3 gpurun_out/bench_v.log | cut -c1-300

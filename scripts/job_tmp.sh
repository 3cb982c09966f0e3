cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
grep -B2 -A25 "Error\|FAIL" gpurun_out/pytest_gpu.log | head -60
echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"
timeout 900 python scripts/cache_study.py --out gpurun_out/cache_study_heap.json --budgets 1000,2500 --slots 1.25,1.5 --heaps layer,global > gpurun_out/cache_study_heap.log 2>&1; cut -c1-200 gpurun_out/cache_study_heap.log | tail -3

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests -m gpu -q -k "global_heap or v_only" 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log
echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"
timeout 900 python scripts/cache_study.py --out gpurun_out/cache_study_heap.json --budgets 1000,2500 --slots 1.25,1.5 --heaps layer,global > gpurun_out/cache_study_heap.log 2>&1; echo "study rc=$?"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/quick_tc.py > gpurun_out/quick.log 2>&1; echo "quick rc=$?"; tail -3 gpurun_out/quick.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
grep -B2 -A25 "Error\|FAIL" gpurun_out/pytest_gpu.log | head -40
for i in 1 2; do echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"; done
timeout 300 python scripts/attn_trace.py > gpurun_out/attn_trace.log 2>&1; tail -7 gpurun_out/attn_trace.log

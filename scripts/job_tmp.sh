cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$i.log 2>&1; tail -1 gpurun_out/pytest_gpu_$i.log; grep FAILED gpurun_out/pytest_gpu_$i.log; done

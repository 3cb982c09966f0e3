cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --local-gpu 0 --steps 2 --warmup 3 --no-cpu > gpurun_out/w2_gloo.log 2>&1; echo "rc=$?"; tail -c 1500 gpurun_out/w2_gloo.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --backend gloo --local-gpu 0 --steps 2 --warmup 3 --no-cpu --cyclic > gpurun_out/w2_gloo_cyclic.log 2>&1; echo "rc=$?"; tail -c 600 gpurun_out/w2_gloo_cyclic.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?"; tail -c 400 gpurun_out/ref.log

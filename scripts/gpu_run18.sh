cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -m gpu -x > gpurun_out/t18.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t18.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --queries 500 --dist-backend gloo > gpurun_out/bench18_2rank.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench18_2rank.log

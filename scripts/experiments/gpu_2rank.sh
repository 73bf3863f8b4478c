# Two ranks on one GPU over gloo: the sharded path end to end (d_best exchange, lexicographic combine).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --queries 1000 --dist-backend gloo --no-cpu-baseline > gpurun_out/r2_c4.log 2>&1; echo "exit=$?" >> gpurun_out/r2_c4.log

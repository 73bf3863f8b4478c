cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b40_k8192.log 2>&1
timeout 600 python bench.py --config C1 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b40_c1a.log 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b40_c2.log 2>&1

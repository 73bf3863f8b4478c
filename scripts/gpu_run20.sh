cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out


timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --no-cpu-baseline > gpurun_out/bench21.log 2>&1

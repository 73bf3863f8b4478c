cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config C1 --window-index 0 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b22_c1a.log 2>&1
timeout 600 python bench.py --config C1 --window-index 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b22_c1b.log 2>&1
timeout 600 python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b22_c2.log 2>&1
timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b22_c3.log 2>&1
timeout 600 python bench.py --config C0 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b22_c0.log 2>&1

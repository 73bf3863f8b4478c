cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2w_tests.log
timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_c3.log 2>&1
timeout 300 python bench.py --config C0 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r2w_c0.log 2>&1
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2w_c1.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_c4.log 2>&1

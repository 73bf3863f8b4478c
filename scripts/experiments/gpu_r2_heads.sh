cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_index.py -m gpu -x -q > gpurun_out/r2h_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2h_tests.log
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c4_1k.log 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c2.log 2>&1
timeout 300 python bench.py --config C1 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c1.log 2>&1
timeout 300 python bench.py --config C1 --window-index 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c1b.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c4.log 2>&1

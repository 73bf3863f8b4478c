cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t23.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t23.log
timeout 600 python bench.py --config C1 --window-index 0 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b23_c1a.log 2>&1
timeout 600 python bench.py --config C1 --window-index 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b23_c1b.log 2>&1
timeout 600 python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b23_c2.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --no-cpu-baseline > gpurun_out/b23_c4.log 2>&1

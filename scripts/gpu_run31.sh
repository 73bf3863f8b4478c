cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or c1b or long_band or edge" > gpurun_out/t31.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t31.log
timeout 600 python bench.py --config C1 --window-index 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b31_c1b.log 2>&1
timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b31_c3.log 2>&1

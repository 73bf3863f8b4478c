cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t20.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t20.log
timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --no-cpu-baseline > gpurun_out/bench20.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t5.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t5.log
timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --method lb_mv --no-cpu-baseline > gpurun_out/bench5.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench5.log
TCDTW_NO_LANE=1 timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --method lb_mv --no-cpu-baseline > gpurun_out/bench5b.log 2>&1

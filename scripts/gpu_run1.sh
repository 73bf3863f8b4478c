cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --durations=15 > gpurun_out/t1.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --method lb_mv --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench1.log

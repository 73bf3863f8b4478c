cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "select_method or gpu_cost or tc_dtw_select" > gpurun_out/auto_tests.log 2>&1; echo "exit=$?" >> gpurun_out/auto_tests.log
for cfg in "C1" "C2" "C3"; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --method auto > gpurun_out/auto_$cfg.log 2>&1
done
timeout 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --queries 1000 --method auto > gpurun_out/auto_C4_1kq.log 2>&1

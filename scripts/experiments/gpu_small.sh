cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/small_tests.log 2>&1; echo "exit=$?" >> gpurun_out/small_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B --config C0 > gpurun_out/small_c0.log 2>&1
TCDTW_NO_SMALL_WAVE=1 timeout 300 $B --config C0 > gpurun_out/small_c0_off.log 2>&1
timeout 300 $B --config C1 > gpurun_out/small_c1a.log 2>&1
timeout 300 $B --config C3 > gpurun_out/small_c3.log 2>&1

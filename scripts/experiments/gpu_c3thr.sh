cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or edge or long_band" > gpurun_out/c3t_tests.log 2>&1; echo "exit=$?" >> gpurun_out/c3t_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3"
TCDTW_WAVE_THREADS=256 timeout 300 $B > gpurun_out/c3t_256.log 2>&1
TCDTW_WAVE_THREADS=384 timeout 300 $B > gpurun_out/c3t_384.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C1 --window-index 1 --method lb_mv > gpurun_out/c3t_c1b.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_properties.py -m gpu -x -q -k "c3 or c0 or edge or long_band or golden or trigger or enumeration" > gpurun_out/wp_tests.log 2>&1; echo "exit=$?" >> gpurun_out/wp_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3"
TCDTW_WAVE_P=1 timeout 300 $B > gpurun_out/wp_c3_p1.log 2>&1
TCDTW_WAVE_P=2 timeout 300 $B > gpurun_out/wp_c3_p2.log 2>&1
TCDTW_WAVE_P=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config C0 > gpurun_out/wp_c0_p1.log 2>&1
TCDTW_WAVE_P=2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config C0 > gpurun_out/wp_c0_p2.log 2>&1

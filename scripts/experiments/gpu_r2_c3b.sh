cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c0 or filter or edge or long or c4" > gpurun_out/r2c3b_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2c3b_tests.log
timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2c3b_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dtw_wave_d|fin_rescore_warp" -s 1 -c 2 -o gpurun_out/r2c3b_ncu python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2c3b_ncu.log 2>&1
echo "ncu exit=$?" >> gpurun_out/r2c3b_ncu.log

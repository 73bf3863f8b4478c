cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c3 or c0 or edge or long_band" > gpurun_out/c3c2_tests.log 2>&1; echo "exit=$?" >> gpurun_out/c3c2_tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/c3c2_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner" -s 1 -c 1 -o gpurun_out/c2_laner python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1

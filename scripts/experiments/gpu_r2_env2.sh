cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "envelope or golden or c0" > gpurun_out/r2e2_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2e2_tests.log
timeout 300 python bench.py --queries 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2e2_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"envelope_vh" -s 1 -c 1 -o gpurun_out/r2e2_env python bench.py --queries 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2e2_ncu.log 2>&1

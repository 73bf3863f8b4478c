# Envelope v4 + wave_d (unroll 2, finite sqrt operands): parity subset and numbers.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index.py -m gpu -x -q -k "envelope or c3 or c0 or edge or long_band or index or reverse" > gpurun_out/e4_tests.log 2>&1; echo "exit=$?" >> gpurun_out/e4_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B --queries 500 > gpurun_out/e4_c4.log 2>&1
timeout 300 $B --config C3 > gpurun_out/e4_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"envelope_stream" -s 2 -c 1 -o gpurun_out/env4 python bench.py --queries 200 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_env4.log 2>&1

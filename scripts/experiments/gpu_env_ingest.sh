# Envelope kernel v2 + ingest/report GPU tests; C4 envelope number; ncu of the compile-time-D wavefront (C3).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_index.py tests/test_gpu_parity.py -m gpu -x -q -k "envelope or ingest or normalize or report or index or reverse" > gpurun_out/ei_tests.log 2>&1; echo "exit=$?" >> gpurun_out/ei_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B --queries 500 > gpurun_out/ei_c4.log 2>&1
TCDTW_ENV_NAIVE=1 timeout 600 $B --queries 500 > gpurun_out/ei_c4_naive.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_wave_d" -s 1 -c 1 -o gpurun_out/c3_waved python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3d.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu_c3d.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"envelope_stream" -s 2 -c 1 -o gpurun_out/env_stream python bench.py --queries 200 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_env.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu_env.log

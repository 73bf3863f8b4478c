# Full GPU suite; envelope v3 number + ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/e3_tests.log 2>&1; echo "exit=$?" >> gpurun_out/e3_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B --queries 500 > gpurun_out/e3_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"envelope_stream" -s 2 -c 1 -o gpurun_out/env3 python bench.py --queries 200 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_env3.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu_env3.log

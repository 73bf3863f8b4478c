cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_properties.py -m gpu -x -q > gpurun_out/r2tc_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2tc_tests.log
for cfg in "C1" "C3" "C2"; do
  timeout 600 python bench.py --config $cfg --method tc_dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2tc_$cfg.log 2>&1
done
timeout 600 python bench.py --queries 1000 --method tc_dtw --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2tc_C4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"advanced" -s 1 -c 2 -o gpurun_out/r2tc_ncu python bench.py --config C1 --method tc_dtw --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2tc_ncu.log 2>&1

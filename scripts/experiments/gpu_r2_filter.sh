# round 2: float32 filter on float64 data (C3/C0), bit-exact normalize, parser
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ingest.py -m gpu -x -q > gpurun_out/r2f_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2f_tests.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c3.log 2>&1
timeout 300 python bench.py --config C0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c0.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_all.log 2>&1; echo "exit=$?" >> gpurun_out/r2f_all.log

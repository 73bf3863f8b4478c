cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c4 or c1 or c2 or edge or overflow" > gpurun_out/r2p_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2p_tests.log
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_c4_1k.log 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_c2.log 2>&1

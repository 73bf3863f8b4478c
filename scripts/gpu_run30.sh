cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tc_dtw_select" > gpurun_out/t30.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t30.log
timeout 1800 python bench.py > gpurun_out/bench30_full.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench30_full.log

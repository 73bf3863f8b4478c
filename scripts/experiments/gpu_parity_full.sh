cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TCDTW_FULL_PARITY=1 timeout 2400 python -m pytest tests/test_gpu_parity_full.py -m gpu -s -q > gpurun_out/parity_full.log 2>&1; echo "exit=$?" >> gpurun_out/parity_full.log

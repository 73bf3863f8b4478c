cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t17.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t17.log
bash scripts/profile.sh

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fix_tests.log 2>&1; echo "exit=$?" >> gpurun_out/fix_tests.log

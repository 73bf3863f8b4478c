cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/props_tests.log 2>&1; echo "exit=$?" >> gpurun_out/props_tests.log

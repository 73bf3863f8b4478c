cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/tf_tests.log 2>&1; echo "exit=$?" >> gpurun_out/tf_tests.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "saturating or edge or f32_filter or c4 or c1" > gpurun_out/adv_tests.log 2>&1; echo "exit=$?" >> gpurun_out/adv_tests.log
tail -30 gpurun_out/adv_tests.log

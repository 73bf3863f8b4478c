cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/t29.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t29.log
timeout 900 python bench.py --steps 1 --warmup 1 --queries 200 --method lb_pc --no-cpu-baseline > gpurun_out/b29_pc.log 2>&1
timeout 900 python bench.py --steps 1 --warmup 1 --queries 200 --method tc_dtw --no-cpu-baseline > gpurun_out/b29_tc.log 2>&1

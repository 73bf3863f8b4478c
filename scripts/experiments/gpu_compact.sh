cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cmp_tests.log 2>&1; echo "exit=$?" >> gpurun_out/cmp_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --queries 2000 > gpurun_out/cmp_c4.log 2>&1

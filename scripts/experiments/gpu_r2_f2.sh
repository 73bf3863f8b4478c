cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2f2_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2f2_tests.log
timeout 300 python bench.py --config C1 --method lb_pc --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f2_c1_pc.log 2>&1
timeout 300 python bench.py --config C1 --method lb_pc --reverse-pc --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f2_c1_pc_rev.log 2>&1
timeout 600 python bench.py --queries 1000 --method lb_pc --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r2f2_c4_pc.log 2>&1
timeout 600 python bench.py --queries 1000 --method lb_pc --reverse-pc --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r2f2_c4_pc_rev.log 2>&1

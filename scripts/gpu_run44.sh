cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t44.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t44.log
timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b44_c4.log 2>&1
timeout 600 python bench.py --config C2 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b44_c2.log 2>&1
timeout 600 python bench.py --config C1 --window-index 1 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b44_c1b.log 2>&1
timeout 600 python bench.py --config C1 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b44_c1a.log 2>&1

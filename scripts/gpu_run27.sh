cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/t27.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t27.log
timeout 600 python bench.py --config C1 --window-index 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b27_c1b.log 2>&1
timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b27_c3.log 2>&1
TCDTW_NO_PIPE=1 timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b27_c3_wave.log 2>&1

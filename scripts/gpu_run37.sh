cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t37.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t37.log
timeout 600 python bench.py --queries 1000 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b37_l4.log 2>&1
TCDTW_NO_CASC=1 timeout 600 python bench.py --queries 1000 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b37_l4_nocasc.log 2>&1
timeout 600 python bench.py --config C1 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b37_c1a.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t42.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t42.log
for rm in 1 2 3 4 6; do
TCDTW_REFILL_MIN=$rm timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b42_rm$rm.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rm in 1 2 4 6 12; do
TCDTW_REFILL_MIN=$rm timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b39_rm$rm.log 2>&1
done

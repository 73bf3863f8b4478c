cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rm in 1 4 8 16; do
  TCDTW_REFILL_MIN=$rm timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --no-cpu-baseline > gpurun_out/bench16_rm$rm.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --queries 1000"
for r in 2 4 6 8; do TCDTW_REFILL_MIN=$r timeout 600 $B > gpurun_out/rf_$r.log 2>&1; done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --queries 1000"
for t in 4 8 16; do TCDTW_THR_EVERY=$t timeout 600 $B > gpurun_out/thr_$t.log 2>&1; done

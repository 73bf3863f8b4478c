cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C2"
timeout 300 $B > gpurun_out/c2ab_casc.log 2>&1
TCDTW_NO_CASC=1 timeout 300 $B > gpurun_out/c2ab_nocasc.log 2>&1
TCDTW_REFILL_MIN=8 timeout 300 $B > gpurun_out/c2ab_refill8.log 2>&1
TCDTW_REFILL_MIN=1 timeout 300 $B > gpurun_out/c2ab_refill1.log 2>&1

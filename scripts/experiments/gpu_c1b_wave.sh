cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C1 --window-index 1"
timeout 300 $B > gpurun_out/cw_laner.log 2>&1
TCDTW_NO_LANE=1 timeout 300 $B > gpurun_out/cw_wave.log 2>&1
TCDTW_SEG_LEN=64 timeout 300 $B > gpurun_out/cw_seg64.log 2>&1

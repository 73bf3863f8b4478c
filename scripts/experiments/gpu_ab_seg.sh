# A/B: lane-kernel segment length on the small configs; ncu capture of the C3 wavefront kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B --config C1 --window-index 1 > gpurun_out/ab_c1b_auto.log 2>&1
TCDTW_SEG_LEN=2048 timeout 300 $B --config C1 --window-index 1 > gpurun_out/ab_c1b_2048.log 2>&1
TCDTW_SEG_LEN=256 timeout 300 $B --config C1 --window-index 1 > gpurun_out/ab_c1b_256.log 2>&1
TCDTW_SEG_LEN=128 timeout 300 $B --config C1 --window-index 1 > gpurun_out/ab_c1b_128.log 2>&1
timeout 300 $B --config C1 > gpurun_out/ab_c1a_auto.log 2>&1
TCDTW_SEG_LEN=2048 timeout 300 $B --config C1 > gpurun_out/ab_c1a_2048.log 2>&1
timeout 300 $B --config C2 > gpurun_out/ab_c2_auto.log 2>&1
timeout 300 $B --config C3 > gpurun_out/ab_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_wave" -s 1 -c 1 -o gpurun_out/c3_wave python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu_c3.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > gpurun_out/p36_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_lane4" -s 1 -c 1 -o gpurun_out/p36_lane4 $CMD2 > gpurun_out/p36_ncu1.log 2>&1
echo "exit=$?" >> gpurun_out/p36_ncu1.log
TCDTW_NO_LANE4=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_lane_kernel" -s 1 -c 1 -o gpurun_out/p36_lane $CMD2 > gpurun_out/p36_ncu2.log 2>&1
echo "exit=$?" >> gpurun_out/p36_ncu2.log

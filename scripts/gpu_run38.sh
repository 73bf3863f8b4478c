cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > gpurun_out/p38_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_lane4|lbmv_matrix" -s 2 -c 2 -o gpurun_out/p38 $CMD2 > gpurun_out/p38_ncu.log 2>&1
echo "exit=$?" >> gpurun_out/p38_ncu.log

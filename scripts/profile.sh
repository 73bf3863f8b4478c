# Profiling recipe (B200_PROFILING.md): plain run, launch list, full capture
# of the dominant kernels.  Outputs land in gpurun_out/; summaries get copied
# into profiles/ by hand.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --queries 500 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_launches.log 2>&1
echo "launches exit=$?" >> gpurun_out/prof_launches.log
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_lane|lbmv_matrix" -s 2 -c 2 -o gpurun_out/prof_full $CMD2 > gpurun_out/prof_full.log 2>&1
echo "full exit=$?" >> gpurun_out/prof_full.log

# round 2: source-level stall attribution of the lane DTW kernel (ncu --set full --import-source on)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > gpurun_out/r2src2_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner" -s 1 -c 1 -o gpurun_out/r2src2_laner $CMD2 > gpurun_out/r2src2_ncu.log 2>&1
echo "ncu exit=$?" >> gpurun_out/r2src2_ncu.log
ls -la gpurun_out/r2src2_laner.ncu-rep

# ncu --set full captures of the dominant search kernels (reduced C4) and the C3 wavefront.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner" -s 1 -c 1 -o gpurun_out/p2_laner $CMD > gpurun_out/p2_laner.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lbmv_matrix" -s 0 -c 1 -o gpurun_out/p2_lbmv $CMD > gpurun_out/p2_lbmv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_wave_d" -s 1 -c 1 -o gpurun_out/p2_c3 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p2_c3.log 2>&1

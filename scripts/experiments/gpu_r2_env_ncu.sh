cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"envelope_vh" -s 1 -c 1 -o gpurun_out/r2e_env python bench.py --queries 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2e_ncu.log 2>&1
echo "ncu exit=$?" >> gpurun_out/r2e_ncu.log

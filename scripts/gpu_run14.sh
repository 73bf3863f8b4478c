cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t14.log 2>&1
echo "pytest exit=$?" >> gpurun_out/t14.log
timeout 900 python bench.py --steps 2 --warmup 1 --queries 1000 --method lb_mv --no-cpu-baseline > gpurun_out/bench14.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench14.log
CMD="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --method lb_mv --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain14.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_lane|lbmv_matrix" -s 2 -c 2 -o gpurun_out/prof14 $CMD > gpurun_out/ncu14.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu14.log

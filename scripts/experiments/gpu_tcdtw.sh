# TC-DTW (tune_params + tc_dtw_select, as the reference CLI) against LB_MV on every config.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "C0" "C1" "C1 --window-index 1" "C2" "C3"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --method tc_dtw > gpurun_out/tc_$tag.log 2>&1
done
timeout 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --queries 1000 --method tc_dtw > gpurun_out/tc_C4_1kq.log 2>&1

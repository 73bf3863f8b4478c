cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in lb_pc lb_ti tc_dtw none; do
  timeout 900 python bench.py --steps 1 --warmup 1 --queries 200 --method $m --no-cpu-baseline > gpurun_out/bench13_$m.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --queries 1000"
for s in 8 16 32; do timeout 600 $B --seeds $s > gpurun_out/sd_$s.log 2>&1; done

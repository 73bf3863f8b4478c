cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
for kb in 18 36 54 72; do TCDTW_ENV_KB=$kb timeout 600 $B --queries 100 > gpurun_out/e6_kb$kb.log 2>&1; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/e6_c3.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b41_pf.log 2>&1
TCDTW_LANE4_NOPF=1 timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b41_nopf.log 2>&1
TCDTW_LANE4_NOPF=1 TCDTW_REFILL_MIN=4 timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b41_nopf_rm4.log 2>&1
TCDTW_LANE4_NOPF=1 TCDTW_REFILL_MIN=12 timeout 600 python bench.py --queries 1000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b41_nopf_rm12.log 2>&1

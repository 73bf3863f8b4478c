cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ti_tests.log 2>&1; echo "exit=$?" >> gpurun_out/ti_tests.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --queries 200 --method lb_ti"
timeout 900 $B > gpurun_out/ti_smem.log 2>&1
TCDTW_TI_GLOBAL_RING=1 timeout 900 $B > gpurun_out/ti_global.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C1 --method lb_ti > gpurun_out/ti_c1.log 2>&1
TCDTW_TI_GLOBAL_RING=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C1 --method lb_ti > gpurun_out/ti_c1_global.log 2>&1

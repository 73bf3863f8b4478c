# round 2: compact UB / per-index planar copy (parity), LB_MV cascade A/B on C4, full C4 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ab_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r2ab_tests.log
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_casc.log 2>&1
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline --no-cascade > gpurun_out/r2ab_nocasc.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_c4.log 2>&1

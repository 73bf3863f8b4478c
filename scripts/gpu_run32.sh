cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/ubench/isa_rates > gpurun_out/isa_rates.log 2>&1
TCDTW_PIPE=1 timeout 600 python bench.py --config C1 --window-index 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b32_c1b_pipe.log 2>&1
TCDTW_PIPE=1 timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b32_c3_pipe.log 2>&1

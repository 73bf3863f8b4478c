cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_index.py -m gpu -x -q -k "envelope or candidate or golden" > gpurun_out/e7_tests.log 2>&1; echo "exit=$?" >> gpurun_out/e7_tests.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --queries 100"
for kb in 36 54 72; do TCDTW_ENV_KB=$kb timeout 600 $B > gpurun_out/e7_kb$kb.log 2>&1; done

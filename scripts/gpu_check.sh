# Health check of a tree: GPU parity suite, smoke, default bench, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/chk_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.log 2>&1; echo "exit=$?" >> gpurun_out/chk_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/chk_smoke.log
timeout 1200 python bench.py > gpurun_out/chk_bench.log 2>&1; echo "exit=$?" >> gpurun_out/chk_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/chk_ref.log 2>&1; echo "exit=$?" >> gpurun_out/chk_ref.log
tail -3 gpurun_out/chk_tests.log; cat gpurun_out/chk_smoke.log; tail -2 gpurun_out/chk_bench.log | cut -c1-400

# New tests (envelope stream, candidate index / reverse bound, C3 parity with wave_d), C3 A/B, C4 reverse-bound A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -m gpu -x -q -k "envelope or reverse or index or c3 or c0 or edge or long_band" > gpurun_out/wr_tests.log 2>&1; echo "exit=$?" >> gpurun_out/wr_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B --config C3 > gpurun_out/wr_c3_d.log 2>&1
TCDTW_WAVE_GENERIC=1 timeout 300 $B --config C3 > gpurun_out/wr_c3_generic.log 2>&1
timeout 600 $B --queries 1000 > gpurun_out/wr_c4_fwd.log 2>&1
timeout 600 $B --queries 1000 --reverse-bound > gpurun_out/wr_c4_rev.log 2>&1
timeout 300 $B --config C2 --reverse-bound > gpurun_out/wr_c2_rev.log 2>&1
timeout 300 $B --config C1 --window-index 1 --reverse-bound > gpurun_out/wr_c1b_rev.log 2>&1

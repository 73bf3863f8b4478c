# Round-2 evidence pass: GPU suite, opt-in full parity, 2-rank sharded bench
# (gloo, one GPU), default bench, launch list and full captures of the
# dominant kernels.  Outputs in gpurun_out/; summaries copied to profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_tests.log 2>&1; echo "exit=$?" >> gpurun_out/fin_tests.log
TCDTW_FULL_PARITY=1 timeout 2400 python -m pytest tests/test_gpu_parity_full.py -m gpu -x -q -s > gpurun_out/fin_parity_full.log 2>&1; echo "exit=$?" >> gpurun_out/fin_parity_full.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --dist-backend gloo --queries 1000 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/fin_2rank_gloo.log 2>&1; echo "exit=$?" >> gpurun_out/fin_2rank_gloo.log
timeout 1200 python bench.py > gpurun_out/fin_bench.log 2>&1; echo "exit=$?" >> gpurun_out/fin_bench.log
CMD="python bench.py --steps 1 --warmup 1 --queries 1000 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_launches.log 2>&1; echo "exit=$?" >> gpurun_out/fin_launches.log
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner|lbmv_matrix" -s 2 -c 2 -o gpurun_out/fin_full $CMD2 > gpurun_out/fin_full.log 2>&1; echo "exit=$?" >> gpurun_out/fin_full.log
timeout 900 $CMD2 > gpurun_out/fin_plain2.log 2>&1

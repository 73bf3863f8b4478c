# round 2: the saturating LB_MV kernel under ncu (reduced C4) + the adversarial parity test
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "saturating or edge or f32_filter" > gpurun_out/satn_tests.log 2>&1; echo "exit=$?" >> gpurun_out/satn_tests.log
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > gpurun_out/satn_plain.log 2>&1; echo "exit=$?" >> gpurun_out/satn_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lbmv_matrix" -s 1 -c 1 -o gpurun_out/satn_lbmv $CMD2 > gpurun_out/satn_ncu.log 2>&1; echo "exit=$?" >> gpurun_out/satn_ncu.log
python scripts/summarize_ncu.py full gpurun_out/satn_lbmv.ncu-rep "$CMD2 (-k lbmv_matrix -s 1 -c 1)" > gpurun_out/satn_lbmv_summary.txt 2>&1
tail -3 gpurun_out/satn_tests.log

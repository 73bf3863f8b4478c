# Round-2 evidence pass: GPU suite, smoke, opt-in full parity, 2-rank sharded
# bench (gloo, one GPU), per-config benches, default bench + reference arm,
# launch list and full captures of the dominant kernels (summarised on the
# box).  Outputs in gpurun_out/fin3_*; summaries are copied to profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=gpurun_out/fin3
timeout 1500 python -m pytest tests -m gpu -x -q > ${P}_tests.log 2>&1; echo "exit=$?" >> ${P}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "exit=$?" >> ${P}_smoke.log
timeout 1200 python bench.py > ${P}_bench.log 2>&1; echo "exit=$?" >> ${P}_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${P}_bench_ref.log 2>&1; echo "exit=$?" >> ${P}_bench_ref.log
for cfg in "C0" "C1" "C1 --window-index 1" "C2" "C3"; do
  tag=$(echo $cfg | sed 's/ --window-index 1/b/')
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > ${P}_bench_$tag.log 2>&1
done
TCDTW_FULL_PARITY=1 timeout 2400 python -m pytest tests/test_gpu_parity_full.py -m gpu -x -q -s > ${P}_parity_full.log 2>&1; echo "exit=$?" >> ${P}_parity_full.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --dist-backend gloo --queries 1000 --steps 2 --warmup 2 --no-cpu-baseline > ${P}_2rank_gloo.log 2>&1; echo "exit=$?" >> ${P}_2rank_gloo.log
CMD="python bench.py --steps 1 --warmup 1 --queries 1000 --no-cpu-baseline"
timeout 900 $CMD > ${P}_plain.log 2>&1; echo "exit=$?" >> ${P}_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_launches.log 2>&1; echo "exit=$?" >> ${P}_launches.log
python scripts/summarize_ncu.py launches ${P}_launches.csv "$CMD" > ${P}_launches_summary.txt 2>&1
CMD2="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
timeout 900 $CMD2 > ${P}_plain2.log 2>&1; echo "exit=$?" >> ${P}_plain2.log
cap() {  # name, kernel regex, launch skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 -o ${P}_$name "$@" > ${P}_${name}.log 2>&1; echo "exit=$?" >> ${P}_${name}.log
  python scripts/summarize_ncu.py full ${P}_$name.ncu-rep "$* (-k $rx -s $skip -c 1)" > ${P}_${name}_summary.txt 2>&1
  rm -f ${P}_$name.ncu-rep
}
cap ncu_laner dtw_laner 1 $CMD2
cap ncu_lbmv lbmv_matrix 1 $CMD2
cap ncu_env envelope_vh 0 $CMD2
cap ncu_c3 dtw_wave_d 1 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline
ls -la gpurun_out | tail -40

# Round-1 measurement pass: GPU parity suite, smoke, per-config benches, full C4
# (ours + reference arm), ncu launch list of a 1000-query C4 command, and one
# `ncu --set full` capture of each dominant kernel (reduced C4; C3 wavefront).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_tests.log 2>&1; echo "exit=$?" >> gpurun_out/fin_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/fin_smoke.log
for cfg in "C0" "C1" "C1 --window-index 1" "C2" "C3"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/fin_$tag.log 2>&1
done
timeout 1500 python bench.py > gpurun_out/fin_C4.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_C4_ref.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 1 --queries 1000 --no-cpu-baseline > gpurun_out/fin_launches.log 2>&1
echo "launches exit=$?" >> gpurun_out/fin_launches.log
CMD="python bench.py --steps 1 --warmup 1 --queries 256 --candidates 200000 --no-cpu-baseline"
# full captures are summarised on the box (the .ncu-rep files would exceed
# gpurun's 64 MiB copy-back limit) and then deleted
cap() {  # name, kernel regex, launch skip, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 -o gpurun_out/$name "$@" > gpurun_out/${name}.log 2>&1
  python scripts/summarize_ncu.py full gpurun_out/$name.ncu-rep "$* (-k $rx -s $skip -c 1)" > gpurun_out/${name}_summary.txt 2>&1
  rm -f gpurun_out/$name.ncu-rep
}
cap fin_laner dtw_laner 1 $CMD
cap fin_lbmv lbmv_matrix 0 $CMD
cap fin_env envelope_stream 0 $CMD
cap fin_c3 dtw_wave_d 1 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline

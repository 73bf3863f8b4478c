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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner" -s 1 -c 1 -o gpurun_out/fin_laner $CMD > gpurun_out/fin_ncu_laner.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lbmv_matrix" -s 0 -c 1 -o gpurun_out/fin_lbmv $CMD > gpurun_out/fin_ncu_lbmv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"envelope_stream" -s 0 -c 1 -o gpurun_out/fin_env $CMD > gpurun_out/fin_ncu_env.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_wave_d" -s 1 -c 1 -o gpurun_out/fin_c3 python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fin_ncu_c3.log 2>&1

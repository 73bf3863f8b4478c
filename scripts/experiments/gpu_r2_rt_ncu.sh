# round 2: ncu --set full of the run-time-band lane kernel on an off-bucket shape (C4-style data, d=6, W=10)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/offbucket_shapes.py 128 6 10"
timeout 600 $CMD > gpurun_out/rtn_plain.log 2>&1; echo "exit=$?" >> gpurun_out/rtn_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dtw_laner" -s 1 -c 1 -o gpurun_out/rtn_laner $CMD > gpurun_out/rtn_ncu.log 2>&1; echo "exit=$?" >> gpurun_out/rtn_ncu.log
python scripts/summarize_ncu.py full gpurun_out/rtn_laner.ncu-rep "$CMD (-k dtw_laner -s 1 -c 1)" > gpurun_out/rtn_laner_summary.txt 2>&1
rm -f gpurun_out/rtn_laner.ncu-rep
cat gpurun_out/rtn_plain.log; cat gpurun_out/rtn_laner_summary.txt

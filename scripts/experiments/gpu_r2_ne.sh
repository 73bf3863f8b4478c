# round 2: norm expansion in the lane DTW kernel -- parity, then A/B on C4 (1k queries) and the other configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ne_tests.log 2>&1; echo "exit=$?" >> gpurun_out/ne_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B --queries 1000 > gpurun_out/ne_c4_1k.log 2>&1
timeout 300 $B --queries 1000 --no-norm-expansion > gpurun_out/ne_c4_1k_off.log 2>&1
for c in C1 C2; do
  timeout 300 $B --config $c > gpurun_out/ne_$c.log 2>&1
  timeout 300 $B --config $c --no-norm-expansion > gpurun_out/ne_${c}_off.log 2>&1
done
timeout 300 $B --config C1 --window-index 1 > gpurun_out/ne_C1b.log 2>&1
timeout 300 $B --config C1 --window-index 1 --no-norm-expansion > gpurun_out/ne_C1b_off.log 2>&1
tail -3 gpurun_out/ne_tests.log
for f in gpurun_out/ne_c4_1k.log gpurun_out/ne_c4_1k_off.log gpurun_out/ne_C1.log gpurun_out/ne_C1_off.log gpurun_out/ne_C2.log gpurun_out/ne_C2_off.log gpurun_out/ne_C1b.log gpurun_out/ne_C1b_off.log; do echo $f; tail -1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d.get('phases_ms'), d.get('roofline',{}).get('frac'))"; done

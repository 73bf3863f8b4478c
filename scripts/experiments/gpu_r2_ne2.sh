# round 2: norm expansion with the sticky cancellation flag -- parity, then A/B per config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -m gpu -x -q > gpurun_out/ne2_tests.log 2>&1; echo "exit=$?" >> gpurun_out/ne2_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B --queries 1000 > gpurun_out/ne2_c4_1k.log 2>&1
for c in C1 C2; do
  timeout 300 $B --config $c > gpurun_out/ne2_$c.log 2>&1
done
timeout 300 $B --config C1 --window-index 1 > gpurun_out/ne2_C1b.log 2>&1
tail -5 gpurun_out/ne2_tests.log
for f in ne2_c4_1k ne2_C1 ne2_C2 ne2_C1b; do echo $f; tail -1 gpurun_out/$f.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['phase_ms']['dtw'], d.get('roofline',{}).get('frac_of_nominal'))"; done

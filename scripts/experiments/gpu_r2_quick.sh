# round 2: quick A/B of a lane-kernel change -- parity tests of the search, then C4 (1k queries), C1b, C2
# usage: gpu_r2_quick.sh TAG
TAG=${1:-q}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "exit=$?" >> gpurun_out/${TAG}_tests.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $B --queries 1000 > gpurun_out/${TAG}_c4_1k.log 2>&1
timeout 300 $B --config C2 > gpurun_out/${TAG}_C2.log 2>&1
timeout 300 $B --config C1 --window-index 1 > gpurun_out/${TAG}_C1b.log 2>&1
tail -4 gpurun_out/${TAG}_tests.log
for f in ${TAG}_c4_1k ${TAG}_C2 ${TAG}_C1b; do echo $f; tail -1 gpurun_out/$f.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['phase_ms']['dtw'], d['counters']['dtw_cells'], d['counters']['cells_issued'], d.get('roofline',{}).get('frac_of_nominal'))"; done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-q2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "exit=$?" >> gpurun_out/${T}_tests.log
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c4_1k.log 2>&1
timeout 300 python bench.py --config C1 --window-index 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_C1b.log 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_C2.log 2>&1
tail -3 gpurun_out/${T}_tests.log
for f in c4_1k C1b C2; do python - <<PY
import json
for l in open("gpurun_out/${T}_$f.log"):
    if l.startswith("{"):
        j=json.loads(l); print("$f", round(j["value"],1), {k:round(v,1) for k,v in j["phase_ms"].items()}, j["roofline"].get("frac_of_nominal"))
PY
done

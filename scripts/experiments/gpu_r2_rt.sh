cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-rt}
timeout 1200 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "exit=$?" >> gpurun_out/${T}_tests.log
tail -5 gpurun_out/${T}_tests.log
timeout 1200 python scripts/offbucket_shapes.py > gpurun_out/${T}_offbucket.txt 2>&1; cat gpurun_out/${T}_offbucket.txt
timeout 300 python bench.py --queries 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c4_1k.log 2>&1
python - <<PY
import json
for l in open("gpurun_out/${T}_c4_1k.log"):
    if l.startswith("{"):
        j=json.loads(l); print("c4_1k", round(j["value"],1), {k:round(v,1) for k,v in j["phase_ms"].items()}, j["roofline"].get("frac_of_nominal"))
PY

# round 2: wide-point lane kernels (d >= 12) without the 128-register cap (5 blocks per SM by launch bounds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shapes.py -m gpu -x -q > gpurun_out/wide_tests.log 2>&1; echo "exit=$?" >> gpurun_out/wide_tests.log
tail -3 gpurun_out/wide_tests.log
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wide_C2.log 2>&1
python - <<PY
import json
for l in open("gpurun_out/wide_C2.log"):
    if l.startswith("{"):
        j=json.loads(l); print("C2", round(j["value"],1), {k:round(v,1) for k,v in j["phase_ms"].items()}, j["roofline"].get("frac_of_nominal"))
PY
for s in "128 12 12" "64 16 6" "64 20 6"; do timeout 300 python scripts/offbucket_shapes.py $s; done

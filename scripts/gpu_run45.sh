cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "C0" "C1" "C1 --window-index 1" "C2" "C3"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/b45_$tag.log 2>&1
done
timeout 1500 python bench.py > gpurun_out/b45_full.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b45_ref.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/bench15_full.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench15_full.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench15_ref.log 2>&1
echo "ref exit=$?" >> gpurun_out/bench15_ref.log

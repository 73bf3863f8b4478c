cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TCDTW_DEBUG=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python -X faulthandler scripts/debug_search.py > gpurun_out/dbg.log 2>&1
echo "exit=$?" >> gpurun_out/dbg.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TCDTW_DEBUG=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/debug_c3.py > gpurun_out/dbg25.log 2>&1
echo "exit=$?" >> gpurun_out/dbg25.log



cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TCDTW_DEBUG=1 timeout 1200 python scripts/debug_pipe.py > gpurun_out/dbg26.log 2>&1

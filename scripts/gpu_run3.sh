cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/cuda-gdb -batch -ex "set pagination off" -ex "break exit" -ex "break _exit" -ex run -ex bt -ex "info sharedlibrary" --args python scripts/debug_search.py > gpurun_out/gdb.log 2>&1
echo "exit=$?" >> gpurun_out/gdb.log

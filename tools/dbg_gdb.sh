cd $GRAFT_REPO_ROOT
timeout 300 /usr/local/cuda/bin/cuda-gdb -batch -ex run -ex bt -ex "info threads" --args python tools/dbg_seg.py ${1:-6} 1 small_box > gpurun_out/gdb.log 2>&1
grep -v "^\[New Thread\|^\[Thread" gpurun_out/gdb.log | tail -40

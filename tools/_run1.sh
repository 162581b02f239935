cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tools/ab.sh ab1 flat seg
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/t1_pytest.log 2>&1; tail -3 gpurun_out/t1_pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -s > gpurun_out/t1_full.log 2>&1; tail -8 gpurun_out/t1_full.log
nproc; free -g | head -2

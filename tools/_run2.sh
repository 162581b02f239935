cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tools/ab.sh ab2 flat seg seg3 seg2
SPFD_SPAN_KERNEL=seg timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/t2_pytest.log 2>&1; tail -3 gpurun_out/t2_pytest.log

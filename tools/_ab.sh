cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_distributed.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/fin_$i.json 2>/dev/null; python tools/show_bench.py gpurun_out/fin_$i.json 2>/dev/null | head -1; done

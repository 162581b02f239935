#!/bin/bash
# A/B of the fine-kernel kinds on C3 (bench lines) + the kernel A/B tests
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-ab}
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
for k in fused pf fused pf; do
  SPFD_SPAN_KERNEL=$k timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_$k.json 2>/dev/null
  python tools/show_bench.py gpurun_out/${tag}_$k.json | head -1
done
python tools/show_bench.py gpurun_out/${tag}_fused.json

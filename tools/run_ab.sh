#!/bin/bash
# A/B of the fine kernels + ncu --set full of the SpMV kernels and the level-1 smoother
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-ab}
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; tail -3 gpurun_out/${tag}_pytest.log
for k in ${KINDS:-flat zm}; do
  SPFD_SPAN_KERNEL=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_$k.json'));print('$k',d['ms_per_step'],d['roofline']['achieved'],d['kernels'])"
done
for k in ${NCU_KINDS:-zm}; do
SPFD_SPAN_KERNEL=$k timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_span|k_zm|k_zt" -c 4 -o gpurun_out/${tag}_full_$k \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_$k.log 2>&1
tail -2 gpurun_out/${tag}_ncu_$k.log
done

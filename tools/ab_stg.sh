#!/bin/bash
# staged kernel (kind 5) vs the default: kernel A/B tests, C3 bench lines, launch lists
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-stg}
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/${tag}_kt.log 2>&1; tail -5 gpurun_out/${tag}_kt.log
for k in stg pf stg pf; do
  SPFD_SPAN_KERNEL=$k timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_$k.json 2>gpurun_out/${tag}_$k.err
  tail -2 gpurun_out/${tag}_$k.err
  python tools/show_bench.py gpurun_out/${tag}_$k.json  2>/dev/null | head -1
done
for k in stg; do
SPFD_SPAN_KERNEL=$k SPFD_PCG_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
     --log-file gpurun_out/${tag}_launches_$k.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/${tag}_launches_$k.csv 14
done

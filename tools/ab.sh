#!/bin/bash
# A/B of the fine-level kernels on C3 (bench lines without the CPU leg) plus
# the kernel / parity GPU tests.  usage: tools/ab.sh tag [kinds...]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-ab}; shift
kinds=${@:-pf flat}
for k in $kinds; do
  SPFD_SPAN_KERNEL=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tol-reps 0 \
     > gpurun_out/${tag}_bench_$k.json 2> gpurun_out/${tag}_bench_$k.err
  python tools/show_bench.py gpurun_out/${tag}_bench_$k.json
done

#!/bin/bash
# A/B of two library builds on C3 (bench lines without the CPU leg): default vs $SPFD_LIB_B
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-lib}; b=${2:-paper_2010_12879_b200/libspfd_b200_m5.so}
for v in a b a b; do
  if [ $v = b ]; then export SPFD_LIB=$PWD/$b; else unset SPFD_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_$v.json 2>/dev/null
  python tools/show_bench.py gpurun_out/${tag}_$v.json 2>/dev/null | head -5
done

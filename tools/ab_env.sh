#!/bin/bash
# A/B of an environment toggle on C3 bench lines: tools/ab_env.sh tag "VAR=a" "VAR=b"
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=$1; A=$2; B=$3
for v in A B A B; do
  if [ $v = A ]; then e=$A; else e=$B; fi
  env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_$v.json 2>/dev/null
  echo "$e"; python tools/show_bench.py gpurun_out/${tag}_$v.json 2>/dev/null | grep -E "ms/step|level1|fine_spmv"
done

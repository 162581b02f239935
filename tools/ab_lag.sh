#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for lag in 600 1200 2400 100000; do
  SPFD_FUSE_LAG=$lag timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/lag_$lag.json 2>/dev/null
  echo "lag $lag"; python tools/show_bench.py gpurun_out/lag_$lag.json 2>/dev/null | grep -E "ms/step|fused"
done

#!/bin/bash
mkdir -p gpurun_out
for g in 0 4 8 16 32; do
  SPFD_CSR_GROUP=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/grp_$g.json 2>/dev/null
done

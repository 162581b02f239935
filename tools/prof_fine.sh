#!/bin/bash
# ncu --set full of the fine SpMV kernel variants (one launch each) on C3
mkdir -p gpurun_out
for k in items flat; do
  SPFD_SPAN_KERNEL=$k timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
     -k regex:"k_items|k_span" -c 6 -o gpurun_out/prof_fine_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_fine_$k.log 2>&1
done

#!/bin/bash
# A/B of the fine-level kernel variants on C3 (bench lines per variant)
mkdir -p gpurun_out
for k in ${@:-flat tile}; do
  SPFD_SPAN_KERNEL=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$k.json 2> gpurun_out/ab_$k.err
  SPFD_SPAN_KERNEL=$k timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stencil or solve or efield" > gpurun_out/ab_$k.pytest 2>&1
done

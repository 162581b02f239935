#!/bin/bash
# ncu --set full (source-level) of the fine SpMV and the level-1 coarse smoother on C3
tag=${1:-ncu}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_span<2, 0|k_csr<8, 2, 1|k_span<2, 4|k_csr<4, 2, 4" -c 4 -o gpurun_out/${tag}_full \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
ls -la gpurun_out/

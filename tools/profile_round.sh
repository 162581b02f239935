#!/bin/bash
# Round evidence: launch list of the bench step + ncu --set full of the
# fine SpMV (dominant roofline kernel) on C3.  Outputs under gpurun_out/.
tag=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
   --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_span|k_csr|k_update|k_xpby|k_agg_sum" -c 14 -o gpurun_out/${tag}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/

#!/bin/bash
# level-1 smoother lane-group sweep (bench step time) + ncu of the level-1 kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 4 8 16 32; do
  SPFD_CSR_GROUP_A1=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A1 group',$g,d['ms_per_step'])"
done
SPFD_PCG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_csr|k_agg_sum" -c 4 -o gpurun_out/l1_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/l1_ncu.log 2>&1
tail -1 gpurun_out/l1_ncu.log

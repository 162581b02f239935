#!/bin/bash
# launch lists of the C3 bench step with every CSR lane-group width forced
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for g in 0 4 8 16 32; do
  SPFD_CSR_GROUP=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('group',$g,d['ms_per_step'])"
  SPFD_CSR_GROUP=$g timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
     --log-file gpurun_out/grp_$g.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done

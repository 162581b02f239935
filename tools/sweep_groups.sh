#!/bin/bash
# Lane-group sweep of the coarse CSR kernels on C3 (bench lines, no CPU leg).
# usage: tools/sweep_groups.sh "VAR=a" "VAR=b" ...   (default: level-2 knobs)
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
run() { env $1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 2>/dev/null > gpurun_out/sw.json; echo "$1 $(python tools/show_bench.py gpurun_out/sw.json 2>/dev/null | head -1 | grep -o 'ms/step [0-9.]*')"; }
if [ $# -eq 0 ]; then
  set -- X=0 SPFD_GROUP_R1=8 SPFD_GROUP_R1=32 SPFD_GROUP_A2=8 SPFD_GROUP_A2=32 SPFD_GROUP_Q2=8 SPFD_GROUP_Q2=32 \
         SPFD_CSR_PF=1 SPFD_GROUP_RSPAN=8 SPFD_GROUP_RSPAN=2 SPFD_GROUP_A1=8 X=0
fi
for v in "$@"; do run "$v"; done

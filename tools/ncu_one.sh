#!/bin/bash
# ncu --set full of one launch of a kernel (regex $2) in a C3 bench step; env passes through
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-one}; kre=${2:-k_span}; skip=${3:-2}
SPFD_PCG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"$kre" --launch-skip $skip -c 1 \
   -o gpurun_out/${tag} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_ncu.log 2>&1
tail -3 gpurun_out/${tag}_ncu.log

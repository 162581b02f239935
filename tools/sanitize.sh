#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py: one log per tool under
# gpurun_out/ (summaries are copied to profiles/ by hand).
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-san}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_case.py > gpurun_out/${tag}_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/${tag}_$tool.log
  if [ $tool = racecheck ] || [ $tool = synccheck ]; then   # the same kernels launched without CUDA graphs
    SPFD_PCG_GRAPH=0 SANITIZE_NO_GRAPHS=1 timeout 1500 $CS --tool $tool --print-limit 50 python tools/sanitize_case.py \
        > gpurun_out/${tag}_${tool}_nographs.log 2>&1
    echo "$tool (no graphs) rc=$?"; tail -3 gpurun_out/${tag}_${tool}_nographs.log
  fi
done

#!/bin/bash
# Round evidence (one GPU call): C3 bench line (with the CPU baseline and the
# 1e-8 / 1e-12 tolerance table), the reference arm, C4 and C5 numbers, the
# launch list of one C3 step, and ncu --set full of the V-cycle / SpMV
# kernels of one PCG iteration.  Outputs under gpurun_out/.
# The launch list and ncu passes run the host-loop PCG (SPFD_PCG_GRAPH=0):
# the same kernels the default graph runs, launched individually so ncu
# attributes them (kernels inside a WHILE-node body are not profiled).
cd ${GRAFT_REPO_ROOT:-.}
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${tag}_c3_bench.json 2> gpurun_out/${tag}_c3_bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${tag}_c3_reference.json 2> gpurun_out/${tag}_c3_reference.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_c4_bench.json 2> gpurun_out/${tag}_c4_bench.err
timeout 900 python tools/bench_streaming.py > gpurun_out/${tag}_c5_measured.json 2> gpurun_out/${tag}_c5.err
timeout 900 python tools/bench_streaming.py --mode uniform > gpurun_out/${tag}_c5_uniform.json 2>> gpurun_out/${tag}_c5.err
SPFD_PCG_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
   --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > /dev/null 2>&1
SPFD_PCG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_span|k_csr|k_update|k_xpby|k_agg_sum" --launch-skip 3 -c 26 -o gpurun_out/${tag}_full \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_ncu.log 2>&1
ls -la gpurun_out/ | grep ${tag}

#!/bin/bash
# GPU tests, smoke, the launch list of one C3 step and ncu --set full of one
# PCG iteration (host loop, so ncu attributes every kernel).  Outputs under gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-r02g}
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_pytest.log 2>&1; tail -2 gpurun_out/${tag}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
SPFD_PCG_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
   --log-file gpurun_out/${tag}_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > /dev/null 2>&1
SPFD_PCG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" \
   -k regex:"k_span|k_csr|k_update|k_xpby|k_agg_sum" --launch-skip 3 -c 26 -o gpurun_out/${tag}_full \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_ncu.log 2>&1
ls gpurun_out | grep $tag

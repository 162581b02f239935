#!/bin/bash
# one C3 bench line (no CPU leg, no tolerance table) + the bench JSON test
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
tag=${1:-q}
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_bench.err
python tools/show_bench.py gpurun_out/${tag}_bench.json
timeout 600 python -m pytest tests/test_gpu_bench.py -q -x 2>&1 | tail -2

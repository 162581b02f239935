#!/bin/bash
# A/B an environment switch on the C3 bench + parity tests: tools/ab_env.sh VAR val1 val2 ...
var=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${var}_$v.json 2> gpurun_out/ab_${var}_$v.err
  env $var=$v timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/ab_${var}_$v.pytest 2>&1
done

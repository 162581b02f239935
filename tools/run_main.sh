#!/bin/bash
# full GPU test suite + bench (graph PCG on/off) + launch list of the default path
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tag=${1:-main}
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_pytest.log 2>&1; tail -3 gpurun_out/${tag}_pytest.log
for gr in 1 0; do
  SPFD_PCG_GRAPH=$gr timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_g$gr.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_g$gr.json'));print('graph=$gr',d['ms_per_step'],d['iterations'],d['roofline']['achieved'],d['gpu_launches'],d['e2e']['value'])"
done
SPFD_PCG_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
     --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/${tag}_launches.csv 30

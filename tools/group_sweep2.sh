#!/bin/bash
# per-level lane-group overrides on the C3 bench step
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*',d['ms_per_step'])"; }
run X=0
run X=0
run SPFD_GROUP_R1=32
run SPFD_GROUP_R1=8
run SPFD_GROUP_A2=8
run SPFD_GROUP_A2=32
run SPFD_GROUP_AP2=8
run SPFD_GROUP_AP2=32
run SPFD_GROUP_AP1=8
run SPFD_GROUP_P0=4
run SPFD_GROUP_R2=64
run SPFD_GROUP_R2=256

#!/bin/bash
# level-1 lane groups with the Morton layout
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*',d['ms_per_step'])"; }
run X=0
run SPFD_GROUP_A1=8
run SPFD_GROUP_AP1=8
run SPFD_GROUP_A1=8 SPFD_GROUP_AP1=8
run SPFD_GROUP_A1=16
run X=0

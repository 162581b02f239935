cd ${GRAFT_REPO_ROOT:-.}
run() { env $1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 2>/dev/null > gpurun_out/sw.json; echo "$1 $(python tools/show_bench.py gpurun_out/sw.json 2>/dev/null | head -1 | grep -o 'ms/step [0-9.]*')"; }
run "X=0"
run "SPFD_GROUP_R1=8"
run "SPFD_GROUP_R1=32"
run "SPFD_GROUP_Q1=8"
run "SPFD_GROUP_Q1=2"
run "SPFD_GROUP_A1=2"
run "SPFD_GROUP_Q2=8"
run "SPFD_GROUP_Q2=32"
run "SPFD_GROUP_A2=8"
run "SPFD_GROUP_A2=32"
run "X=0"

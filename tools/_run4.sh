cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tools/ab.sh ab4 flat pf
SPFD_CSR_PF=1 SPFD_SPAN_KERNEL=flat timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/ab4_bench_csrpf.json 2>/dev/null
python tools/show_bench.py gpurun_out/ab4_bench_csrpf.json
SPFD_CSR_PF=1 SPFD_SPAN_KERNEL=pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/ab4_bench_both.json 2>/dev/null
python tools/show_bench.py gpurun_out/ab4_bench_both.json

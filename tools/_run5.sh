cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for a in 0 148 444 888; do
  SPFD_PF_AHEAD=$a SPFD_SPAN_KERNEL=pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/ab5_pf$a.json 2>/dev/null
  echo "ahead=$a"; python tools/show_bench.py gpurun_out/ab5_pf$a.json
done
SPFD_SPAN_KERNEL=pf SPFD_PCG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none \
   -k regex:"k_span" --launch-skip 20 -c 5 -o gpurun_out/ab5_pf_full \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tol-reps 0 --kernel-reps 2 > gpurun_out/ab5_ncu.log 2>&1
tail -3 gpurun_out/ab5_ncu.log

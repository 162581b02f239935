cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rv in 1 0 1 0; do
  SPFD_REV=$rv timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tol-reps 0 > gpurun_out/ab_rev$rv.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_rev$rv.json'));print('rev=$rv',d['ms_per_step'],d['iterations'],d['e2e']['value'])"
done
timeout 900 python -m pytest tests -q -m gpu -x -k "not fullsize" 2>&1 | tail -3

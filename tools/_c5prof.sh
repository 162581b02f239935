cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_field.py tests/test_gpu_pipeline.py -x -q -m gpu 2>&1 | tail -3
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dgemm|k_sub_div|k_lap" --csv --log-file gpurun_out/c5_gemm_mma3.csv python tools/bench_streaming.py --count 2 > /dev/null 2>&1
timeout 600 python tools/bench_streaming.py --count 100 > gpurun_out/c5_after5.json 2>/dev/null; cat gpurun_out/c5_after5.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['per_snapshot_ms_mean'], d['stage_ms_mean'])"

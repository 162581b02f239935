cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_field.py tests/test_gpu_kernels.py -q -x > gpurun_out/t7_pytest.log 2>&1; tail -3 gpurun_out/t7_pytest.log
timeout 900 python tools/bench_streaming.py > gpurun_out/t7_c5.json 2> gpurun_out/t7_c5.err; python -c "
import json; d=json.loads(open('gpurun_out/t7_c5.json').read().strip().splitlines()[-1]); print(d['per_snapshot_ms_mean'], d['stage_ms_mean'], d['clean_iterations_mean'])"; tail -3 gpurun_out/t7_c5.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t7_bench.json 2> gpurun_out/t7_bench.err; grep bench gpurun_out/t7_bench.err; python tools/show_bench.py gpurun_out/t7_bench.json
bash tools/sanitize.sh r02

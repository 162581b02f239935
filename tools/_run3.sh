cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/t3_pytest.log 2>&1; tail -5 gpurun_out/t3_pytest.log
timeout 900 python bench.py > gpurun_out/t3_bench.json 2> gpurun_out/t3_bench.err; tail -3 gpurun_out/t3_bench.err; python tools/show_bench.py gpurun_out/t3_bench.json
timeout 900 python tools/bench_streaming.py > gpurun_out/t3_c5.json 2> gpurun_out/t3_c5.err; tail -c 1500 gpurun_out/t3_c5.json; tail -3 gpurun_out/t3_c5.err
timeout 1200 python bench.py --impl reference > gpurun_out/t3_ref.json 2> gpurun_out/t3_ref.err; tail -c 600 gpurun_out/t3_ref.json

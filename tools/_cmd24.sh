timeout 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -1
timeout 120 python tools/probe_latency.py --label rel --batches 4,8 2>&1 | cut -c1-160
timeout 600 python bench.py --no-cpu > gpurun_out/bench_v13.log 2>&1; tail -1 gpurun_out/bench_v13.log | cut -c1-100

timeout 500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/sweep.py --which 3,4 --out gpurun_out/sweep34_v11.jsonl > /dev/null 2>&1; wc -l gpurun_out/sweep34_v11.jsonl
timeout 600 python bench.py > gpurun_out/bench_v11.log 2>&1; tail -1 gpurun_out/bench_v11.log | cut -c1-120

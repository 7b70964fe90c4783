timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
O=gpurun_out/lat17.jsonl; rm -f $O
timeout 120 python tools/probe_latency.py --label v8 --batches 1,2,4,8 --out $O
ALAYA_TC_BALANCE=0 timeout 120 python tools/probe_latency.py --label v8_nobal --batches 1,2,4,8 --out $O
cut -c1-140 $O

timeout 900 python tools/sweep.py --which 3,4 --out gpurun_out/sweep34_v7.jsonl > gpurun_out/sweep34.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"alaya|scan_tc" -c 200 --csv --log-file gpurun_out/launches_v7.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scan_tc_kernel|attend_ovl_kernel" -s 6 -c 2 -o gpurun_out/ncu_v7 python bench.py --steps 1 --warmup 1 --layers 4 --no-cpu --no-e2e --profile > /dev/null 2>&1
ls -la gpurun_out

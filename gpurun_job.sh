timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > /dev/null 2>&1
grep -i "transpose\|memset" gpurun_out/launches_t.csv | cut -c1-200 | head -5

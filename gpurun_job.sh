for i in 1 2 3; do timeout 300 python tools/fit_bench.py 1000 10 50 1 2>&1 | tail -2; done
nproc; cat /proc/loadavg

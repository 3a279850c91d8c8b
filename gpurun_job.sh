mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-200
timeout 300 python bench.py --n 100000 --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_1e5.json 2>/dev/null
timeout 600 python bench.py --n 10000000 --steps 10 --warmup 3 --no-cpu --e2e-steps 4 > gpurun_out/bench_1e7.json 2>/dev/null
timeout 900 python bench.py --n 1000000 --p 1000 --m 1000 --steps 10 --warmup 3 --no-cpu --e2e-steps 4 > gpurun_out/bench_cfg5.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>/dev/null
timeout 300 python tools/fit_bench.py 1000 10 50 1 > gpurun_out/fit_cfg1.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 3 -c 1 -o gpurun_out/sweep_full python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 200 python tools/timeline.py 1000000 100 200 > gpurun_out/timeline_1e6.txt 2>&1
timeout 200 python tools/timeline.py 100000 100 200 > gpurun_out/timeline_1e5.txt 2>&1
timeout 300 python tools/multichain_bench.py 100000 4 200 > gpurun_out/multichain.txt 2>&1
for f in bench bench_1e5 bench_1e7 bench_cfg5 bench_ref; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d.get('e2e',{}).get('value'))"; done; cat gpurun_out/fit_cfg1.txt

mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for n in 300000 1000000 100000; do timeout 60 python tools/timeline.py $n 100 200 > gpurun_out/timeline_$n.txt 2>&1; cat gpurun_out/timeline_$n.txt; done
timeout 200 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json

mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 200 python tools/timeline.py 1e6 100 200 > gpurun_out/timeline_1e6.txt 2>&1; cat gpurun_out/timeline_1e6.txt
timeout 200 python tools/timeline.py 1e5 100 200 > gpurun_out/timeline_1e5.txt 2>&1; cat gpurun_out/timeline_1e5.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json

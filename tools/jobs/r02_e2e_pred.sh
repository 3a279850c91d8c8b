#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/e2e_timing.py 200 > gpurun_out/e2e_timing.txt 2>&1; cat gpurun_out/e2e_timing.txt | tail -6
for a in "10000 500" "100000 200" "1000000 50"; do timeout 300 python tools/predict_bench.py $a 2>&1 | tail -1; done | tee gpurun_out/predict_bench.txt

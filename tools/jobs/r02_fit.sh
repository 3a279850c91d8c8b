#!/bin/bash
mkdir -p gpurun_out
for a in "1000 10 50 1" "100000 100 200 1" "100000 100 200 2" "1000000 100 200 1" "1000000 100 200 2"; do
  timeout 600 python tools/fit_bench.py $a 2>&1 | grep "^fit"
done | tee gpurun_out/fit_bench.txt

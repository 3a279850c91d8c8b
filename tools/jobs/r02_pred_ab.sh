#!/bin/bash
for lib in base0 cur; do
  if [ $lib = cur ]; then unset BART_LIB; else export BART_LIB=paper_2410_23244_b200/lib/variants/$lib.so; fi
  for a in "10000 500" "100000 200" "1000000 50" "10000 50"; do echo -n "$lib: "; timeout 300 python tools/predict_bench.py $a 2>&1 | tail -1; done
done

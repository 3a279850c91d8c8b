#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_forest_shapes.py tests/test_gpu_parity.py tests/test_gpu_fit.py -q -k "forest or evaluate or traverse or fit or stream_mode_large" 2>&1 | tail -2
for v in trav_old cur trav_old cur; do
  if [ $v = cur ]; then unset BART_LIB; else export BART_LIB=paper_2410_23244_b200/lib/variants/$v.so; fi
  echo -n "$v: "; timeout 300 python tools/forest_profile.py 200 20 2>&1 | tail -1
done

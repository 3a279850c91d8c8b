#!/bin/bash
# fused-evaluate variants: parity (in-tree lib) + per-launch times on a burned-in chain
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_forest_shapes.py tests/test_gpu_parity.py -k "forest or evaluate" -x -q > gpurun_out/pytest_eval.log 2>&1; tail -3 gpurun_out/pytest_eval.log
for v in "$@"; do
  if [ "$v" = base ]; then unset BART_LIB; else export BART_LIB=paper_2410_23244_b200/lib/variants/$v.so; fi
  echo -n "$v: "; timeout 300 python tools/forest_profile.py 200 20 2>&1 | tail -1
done

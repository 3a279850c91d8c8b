#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_shapes.py -x -q -k "stream or two_level or ragged or multi_cta or golden" > gpurun_out/pytest_units.log 2>&1; tail -3 gpurun_out/pytest_units.log
for n in 10000000 4000000; do
  timeout 900 python tools/variants.py bench base0 units -- --e2e-steps 5 --n $n --steps 30
done
timeout 900 python tools/variants.py bench base0 units -- --e2e-steps 5 --n 10000000 --steps 30

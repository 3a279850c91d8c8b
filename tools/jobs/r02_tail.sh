#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_shapes.py -x -q 2>&1 | tail -2
for r in 1 2; do
  timeout 900 python tools/variants.py bench tail0 tail1 -- --e2e-steps 10
done
timeout 900 python tools/variants.py bench tail0 tail1 -- --e2e-steps 10 --n 100000

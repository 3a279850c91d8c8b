#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_swar.log 2>&1; tail -3 gpurun_out/pytest_swar.log
for r in 1 2; do
  timeout 900 python tools/variants.py bench base0 swar -- --e2e-steps 10
done
timeout 900 python tools/variants.py bench base0 swar -- --e2e-steps 10 --n 100000

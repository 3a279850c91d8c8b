#!/bin/bash
# A/B of experiment variants (lib/variants/*.so): headline and n=1e5, alternating
mkdir -p gpurun_out
V="$@"
for r in 1 2; do
  timeout 900 python tools/variants.py bench $V -- --e2e-steps 10
  timeout 900 python tools/variants.py bench $V -- --e2e-steps 10 --n 100000
done

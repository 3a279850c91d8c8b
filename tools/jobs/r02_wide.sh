#!/bin/bash
for r in 1 2; do
  timeout 900 python tools/variants.py bench w0 w1 w2 -- --e2e-steps 10
done
timeout 900 python tools/variants.py bench w0 w1 w2 -- --e2e-steps 10 --n 100000

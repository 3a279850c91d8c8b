#!/bin/bash
for r in 1 2; do timeout 900 python tools/variants.py bench t0 t1 -- --e2e-steps 5; done
timeout 1500 python tools/variants.py bench t0 t1 -- --e2e-steps 5 --p 1000 --m 1000 --steps 20

#!/bin/bash
timeout 1200 python tools/variants.py bench t0 t1 t2 t3 -- --e2e-steps 5
timeout 1500 python tools/variants.py bench t0 t1 t2 t3 -- --e2e-steps 5 --p 1000 --m 1000 --steps 20
timeout 1200 python tools/variants.py bench t0 t1 t2 t3 -- --e2e-steps 5

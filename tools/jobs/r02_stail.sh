#!/bin/bash
timeout 900 python tools/variants.py bench st0 st1 -- --e2e-steps 5 --n 10000000 --steps 30
timeout 900 python tools/variants.py bench st0 st1 -- --e2e-steps 5 --n 10000000 --steps 30

#!/bin/bash
timeout 1200 python tools/variants.py bench c0 c1 c2 -- --e2e-steps 5
timeout 1500 python tools/variants.py bench c0 c1 c2 -- --e2e-steps 5 --p 1000 --m 1000 --steps 20
timeout 1200 python tools/variants.py bench c0 c1 c2 -- --e2e-steps 5

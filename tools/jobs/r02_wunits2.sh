#!/bin/bash
for uw in 128 256 64; do
  echo "unit_words=$uw"
  BART_UNIT_WORDS=$uw timeout 900 python tools/variants.py bench wunits -- --e2e-steps 5 --n 10000000 --steps 30
done
timeout 900 python tools/variants.py bench base0 -- --e2e-steps 5 --n 10000000 --steps 30
BART_UNIT_WORDS=128 timeout 900 python tools/variants.py bench wunits -- --e2e-steps 5 --n 4000000 --steps 30
timeout 900 python tools/variants.py bench base0 -- --e2e-steps 5 --n 4000000 --steps 30

timeout 1500 python tools/variants.py bench v11 bo32 bo100 bo250 v11 -- --steps 200 --warmup 5 --e2e-steps 2 --no-cpu
timeout 900 python tools/variants.py bench v11 bo32 bo100 -- --n 100000 --steps 300 --warmup 5 --e2e-steps 2 --no-cpu

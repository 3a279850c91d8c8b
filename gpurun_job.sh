timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 python tools/variants.py bench s1 base s1 base -- --n 10000000 --steps 10 --warmup 3 --e2e-steps 2
timeout 900 python tools/variants.py bench s1 base -- --n 3000000 --steps 20 --warmup 3 --e2e-steps 2

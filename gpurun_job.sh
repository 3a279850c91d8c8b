timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 python tools/variants.py bench v10 base nopersist noevict -- --n 10000000 --steps 10 --warmup 3 --e2e-steps 2
timeout 900 python tools/variants.py bench v10 base -- --steps 100 --warmup 5 --e2e-steps 2

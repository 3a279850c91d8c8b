timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 python tools/variants.py bench v11 base v11 base -- --steps 200 --warmup 5 --e2e-steps 2
timeout 900 python tools/variants.py bench v11 base -- --n 100000 --steps 300 --warmup 5 --e2e-steps 2

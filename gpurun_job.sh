timeout 900 env BART_LIB=paper_2410_23244_b200/lib/variants/roles.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 900 python tools/variants.py bench v12 roles v12 roles -- --steps 200 --warmup 5 --e2e-steps 2 --no-cpu
timeout 900 python tools/variants.py bench v12 roles -- --n 100000 --steps 300 --warmup 5 --e2e-steps 2 --no-cpu

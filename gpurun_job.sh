timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python tools/variants.py bench v10 base v10 base -- --steps 200 --warmup 5 --e2e-steps 2

timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['roofline']['kernel_ms'],4))"; done
timeout 200 python bench.py --n 100000 --steps 200 --warmup 5 --no-cpu --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench 1e5', round(d['value'],1), round(d['roofline']['kernel_ms'],4))"
timeout 60 python tools/timeline.py 1000000 100 200 2>&1 | head -16

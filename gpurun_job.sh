timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --e2e-steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['roofline']['kernel_ms'],4), round(d['roofline']['propose_ms'],4))"; done

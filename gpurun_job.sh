timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['forest_kernels']))"

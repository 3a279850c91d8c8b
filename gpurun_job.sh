timeout 300 python bench.py --no-cpu --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('before ref', d['value'], d['e2e']['value'])"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('after ref', d['value'], d['e2e']['value'])"
timeout 300 python tools/fit_bench.py 1000 10 50 1 2>&1 | tail -2
ps aux --sort=-%cpu | head -5

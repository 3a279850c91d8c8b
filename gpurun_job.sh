timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu > gpurun_out/bench_fk.json 2>gpurun_out/bench_fk.err; python -c "
import json; d=json.load(open('gpurun_out/bench_fk.json')); print(d['value']); print(json.dumps(d['forest_kernels'], indent=1))"; tail -3 gpurun_out/bench_fk.err

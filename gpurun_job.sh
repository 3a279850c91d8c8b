mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_cta" > gpurun_out/pytest_mc.log 2>&1; tail -3 gpurun_out/pytest_mc.log
for cfg in "100000 4" "100000 2" "1000000 2" "1000000 4" "10000 8"; do timeout 300 python tools/multichain_bench.py $cfg 200 2>&1 | tail -5; done > gpurun_out/multichain.txt
cat gpurun_out/multichain.txt

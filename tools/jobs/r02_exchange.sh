mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_errors.py -q -x > gpurun_out/pytest_x.log 2>&1; tail -2 gpurun_out/pytest_x.log
timeout 900 python -m pytest tests/test_gpu_ipc_shards.py -q -x > gpurun_out/pytest_ipc.log 2>&1; tail -2 gpurun_out/pytest_ipc.log
./tools/bin/xshard_bench > gpurun_out/xshard_bench.txt 2>&1; cat gpurun_out/xshard_bench.txt
timeout 600 python tools/exchange_emulation.py > gpurun_out/exchange_emulation.txt 2>&1; cat gpurun_out/exchange_emulation.txt

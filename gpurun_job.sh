mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serialize.py tests/test_gpu_fit.py -x -q > gpurun_out/pytest_ser.log 2>&1; tail -25 gpurun_out/pytest_ser.log

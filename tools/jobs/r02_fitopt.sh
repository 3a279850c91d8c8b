#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fit.py tests/test_gpu_serialize.py -x -q 2>&1 | tail -2
for r in 0 1 0 1; do echo "BART_D2H_REGISTER=$r"; BART_D2H_REGISTER=$r timeout 600 python tools/fit_profile.py 1e6 1 2>&1 | grep -E "^fit|trace_read|inverse|stack|quantize|_device_ranges"; done
for r in 1; do BART_D2H_REGISTER=$r timeout 600 python tools/fit_profile.py 1e6 2 2>&1 | grep -E "^fit|trace_read|inverse|stack"; done

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_binning.py tests/test_gpu_fit.py tests/test_cabi.py -x -q 2>&1 | tail -2
for r in 1 2; do timeout 600 python tools/fit_profile.py 1e6 1 2>&1 | grep -E "^fit|trace_read|inverse|quantize|_device_ranges"; done

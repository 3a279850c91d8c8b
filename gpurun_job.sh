mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; tail -3 gpurun_out/pytest_parity.log
timeout 900 python tools/variants.py bench pre_ctrl early plane base pre_ctrl early plane base -- --steps 200 --warmup 5 --e2e-steps 2 > gpurun_out/var.txt 2>&1
timeout 600 python tools/variants.py bench pre_ctrl base -- --n 100000 --steps 300 --warmup 5 --e2e-steps 2 >> gpurun_out/var.txt 2>&1
cat gpurun_out/var.txt

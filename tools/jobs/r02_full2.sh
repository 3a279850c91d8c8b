mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_smoke.py > gpurun_out/racecheck.txt 2>&1; tail -5 gpurun_out/racecheck.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/memcheck.txt 2>&1; tail -3 gpurun_out/memcheck.txt

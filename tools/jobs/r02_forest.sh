mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "forest or evaluate or traverse or fit or posterior or serialize or ragged or golden" > gpurun_out/pytest_forest.log 2>&1; tail -2 gpurun_out/pytest_forest.log
python tools/variants.py bench base notma base -- --steps 20 --e2e-steps 2

timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/timeline.py 1e6 100 200 2>&1 | tail -9
timeout 300 python tools/timeline.py 1e5 100 200 2>&1 | tail -9

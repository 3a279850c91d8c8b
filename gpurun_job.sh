timeout 200 python tools/timeline.py 100000 100 200 2>&1 | head -30
timeout 200 python tools/timeline.py 1000000 100 200 2>&1 | head -8

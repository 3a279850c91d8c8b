timeout 300 python tools/predict_bench.py 100000 200 200 2>&1 | tail -1
BART_LIB=paper_2410_23244_b200/lib/variants/v11.so timeout 300 python tools/predict_bench.py 100000 200 200 2>&1 | tail -1
timeout 300 python tools/predict_bench.py 1000000 50 200 2>&1 | tail -1
timeout 300 python tools/predict_bench.py 10000 500 200 2>&1 | tail -1
BART_LIB=paper_2410_23244_b200/lib/variants/v11.so timeout 300 python tools/predict_bench.py 10000 500 200 2>&1 | tail -1

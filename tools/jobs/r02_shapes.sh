mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_errors.py tests/test_gpu_parity_shapes.py -x -q > gpurun_out/pytest_new.log 2>&1; tail -3 gpurun_out/pytest_new.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_burn.json 2> gpurun_out/bench_burn.err; tail -1 gpurun_out/bench_burn.json | cut -c1-300
for b in 20 300; do BART_TL_BURN=$b timeout 300 python tools/timeline.py 1e6 100 200 > gpurun_out/timeline_burn$b.txt 2>&1; done
head -3 gpurun_out/timeline_burn300.txt

# Round validation on one B200 (run through gpurun): GPU tests, the bench lines
# (headline + the other BASELINE configs), the reference arm, the ncu launch
# list and a full capture of the sweep at steady state (after the 2000-iteration
# burn-in), the per-phase timeline.  Summarise with tools/profile_summary.py TAG.
mkdir -p gpurun_out
rm -f gpurun_out/bench*.json gpurun_out/timeline_*.txt gpurun_out/launches.csv gpurun_out/sweep_full.ncu-rep
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 600 python bench.py --n 100000 --no-cpu > gpurun_out/bench_1e5.json 2>/dev/null
timeout 900 python bench.py --n 10000000 --steps 20 --no-cpu > gpurun_out/bench_1e7.json 2>/dev/null
timeout 1200 python bench.py --p 1000 --m 1000 --steps 20 --no-cpu > gpurun_out/bench_cfg5.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep -s 2003 -c 1 -o gpurun_out/sweep_full python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/ncu_full.log 2>&1
BART_TL_BURN=2000 timeout 300 python tools/timeline.py 1e6 100 200 > gpurun_out/timeline_1e6_burn2000.txt 2>&1
ls gpurun_out

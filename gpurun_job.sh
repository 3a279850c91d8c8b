mkdir -p gpurun_out
./tools/bin/microbench > gpurun_out/microbench.txt 2>&1
timeout 300 python tools/timeline.py 1e6 100 200 > gpurun_out/timeline_1e6.txt 2>&1
timeout 300 python tools/timeline.py 1e5 100 200 > gpurun_out/timeline_1e5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep -s 3 -c 1 -o gpurun_out/sweep_full python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/microbench.txt gpurun_out/timeline_1e6.txt gpurun_out/timeline_1e5.txt; tail -3 gpurun_out/ncu_full.log

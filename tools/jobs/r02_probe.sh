mkdir -p gpurun_out
./tools/bin/l2_near_far > gpurun_out/l2_near_far.txt 2>&1; cat gpurun_out/l2_near_far.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/sanitize_smoke.py > gpurun_out/racecheck_analysis.txt 2>&1; grep -v "^=========     Host\|Saved host" gpurun_out/racecheck_analysis.txt | tail -40

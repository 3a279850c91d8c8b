#!/bin/bash
mkdir -p gpurun_out
for v in sw_k4p2 sw_k8p1 sw_k8p2 sw_k4p1 sw_k4p2; do
  export BART_LIB=paper_2410_23244_b200/lib/variants/$v.so
  echo -n "$v: "; timeout 300 python tools/forest_profile.py 200 20 2>&1 | tail -1
done
export BART_LIB=paper_2410_23244_b200/lib/variants/sw_k4p2.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"evaluate|traverse" -s 4 -c 2 -f -o gpurun_out/ncu_sw_k4p2 python tools/forest_profile.py 200 3 > gpurun_out/ncu_sw.log 2>&1; tail -1 gpurun_out/ncu_sw.log

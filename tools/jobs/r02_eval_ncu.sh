#!/bin/bash
# ncu --set full of the fused evaluate kernel, per variant (lib/variants/NAME.so)
mkdir -p gpurun_out
for v in "$@"; do
  export BART_LIB=paper_2410_23244_b200/lib/variants/$v.so
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:evaluate -s 2 -c 1 -f -o gpurun_out/ncu_$v python tools/forest_profile.py 200 3 > gpurun_out/ncu_$v.log 2>&1
  tail -2 gpurun_out/ncu_$v.log
done

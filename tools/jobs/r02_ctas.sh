#!/bin/bash
# CTA-count sweep of the steady-state step (bench.py --max-ctas), n=1e5 and n=1e6
mkdir -p gpurun_out
python -m paper_2410_23244_b200._build > gpurun_out/build.log 2>&1
run() {  # n ctas [extra]
  local n=$1 c=$2; shift 2
  timeout 300 python bench.py --no-cpu --n $n --max-ctas $c --e2e-steps 10 "$@" > gpurun_out/ctas_${n}_${c}.json 2> gpurun_out/ctas_${n}_${c}.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/ctas_${n}_${c}.json').read().strip().splitlines()[-1])
print('n=$n ctas=%4d  %8.1f it/s  chunk %d  leaves %.2f' % (d['sweep_grid']['ctas'], d['value'], d['sweep_grid']['chunk'], d['trees']['mean_leaves']))" || tail -3 gpurun_out/ctas_${n}_${c}.err
}
for c in 148 128 112 96 80 74 64 48 37; do run 100000 $c; done
for c in 148 132 120 100 80; do run 1000000 $c; done
for c in 148 120 96; do run 1000000 $c --p 1000 --m 1000 --burn 50; done

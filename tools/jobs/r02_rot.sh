#!/bin/bash
# which CTAs publish late at n=1e7 (stream mode) when CTA c sweeps chunk (c + ROT) % 148
mkdir -p gpurun_out
for rot in "" "BART_CHUNK_ROT=27" "BART_CHUNK_ROT=74"; do
  echo "== rot: $rot"
  BART_TL_DEFINES="$rot" BART_TL_BURN=100 timeout 900 python tools/timeline.py 1e7 > gpurun_out/tl_rot_$rot.txt 2>&1
  grep -A 9 "tree period\|latest 8" gpurun_out/tl_rot_$rot.txt | grep -v "^--" | head -14
done

#!/bin/bash
for v in "$@"; do
  export BART_LIB=paper_2410_23244_b200/lib/variants/$v.so
  echo -n "$v: "; timeout 300 python tools/forest_profile.py 200 20 2>&1 | tail -1
done

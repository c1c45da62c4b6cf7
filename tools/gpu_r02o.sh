#!/bin/bash
for spec in "4 256 2048 1024" "13 256 2048 1024"; do
  set -- $spec
  echo "== force $1 shape $2 $3 $4 planes, graph of 20"
  PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $1 --shape $2 $3 $4 --planes --graph 20 2>&1 | tail -20
done

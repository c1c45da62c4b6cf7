#!/bin/bash
for e in 55 23; do
  echo "== PFB_TC_EXP=$e"
  PFB_TC_EXP=$e PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force 4 --shape 256 2048 1024 --planes --graph 20 2>&1 | grep "deltas\|rep 2" | tail -2
done

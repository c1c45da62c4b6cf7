#!/bin/bash
# GEMM path probe for cfg4's per-step shapes (replayed-graph device time)
OUT=gpurun_out/r02b; mkdir -p $OUT
for shp in "256 2048 1024" "256 1024 2048" "256 512 2048" "256 2048 512"; do
  for f in 3 4 7 8 9 5 6 1 10 11; do
    timeout 60 python tools/gemm_probe.py --graph --force $f --shape $shp --iters 40 2>&1 | tail -1
  done
done > $OUT/probe.txt
cat $OUT/probe.txt
for f in 4 7 8 9; do PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $f --shape 256 2048 1024; done > $OUT/trace.txt 2>&1
cat $OUT/trace.txt

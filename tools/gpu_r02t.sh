#!/bin/bash
# per-step cfg4 GEMM shapes: path timings and phase traces
OUT=gpurun_out/r02t; mkdir -p $OUT
for shp in "256 2048 1024" "256 2048 512" "256 512 2048" "16384 2048 512"; do
  for f in 3 4 9 12 13 15 16 17 5 6; do
    echo "shape $shp force $f: $(timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 20 2>&1 | tail -1)"
  done
done > $OUT/probe.txt 2>&1
cat $OUT/probe.txt
for shp in "256 2048 1024" "256 512 2048"; do
 for f in 13 17; do
  echo "== trace $shp force $f"
  PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $f --shape $shp --planes --graph 20 2>&1 | grep -A20 "rep 2"
 done
done > $OUT/trace.txt 2>&1
cat $OUT/trace.txt

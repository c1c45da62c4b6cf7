#!/bin/bash
# GEMM probe: cfg4 per-step shapes (and the K=512 hoisted forward) by path and k-split
OUT=gpurun_out/r02i; mkdir -p $OUT
for shp in "256 2048 1024" "256 2048 512" "256 512 2048"; do
  for f in 4 9 5 6; do
    timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 40 2>&1 | tail -1
  done
  for ks in 1 2 4 8; do
    echo "ksplit=$ks"; PFB_TC_KSPLIT=$ks timeout 60 python tools/gemm_probe.py --graph --planes --force 4 --shape $shp --iters 40 2>&1 | tail -1
    PFB_TC_KSPLIT=$ks timeout 60 python tools/gemm_probe.py --graph --planes --force 3 --shape $shp --iters 40 2>&1 | tail -1
  done
done > $OUT/probe.txt 2>&1
cat $OUT/probe.txt
for ks in 2 4 8; do PFB_TC_KSPLIT=$ks PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force 4 --shape 256 2048 1024 2>&1 | tail -14; done

#!/bin/bash
# GEMM experiment: TMEM chunk depth x k-split x products (1 = hi*hi only, timing only)
OUT=gpurun_out/r02m; mkdir -p $OUT
for shp in "256 2048 1024" "256 512 2048"; do
  for pr in 3 1; do
    for ch in 2 4 8; do
      for ks in 2 4 8; do
        r=$(PFB_TC_PRODUCTS=$pr PFB_TC_CHUNK=$ch PFB_TC_KSPLIT=$ks timeout 60 python tools/gemm_probe.py --graph --planes --force 4 --shape $shp --iters 40 2>&1 | tail -1)
        echo "prod=$pr chunk=$ch ks=$ks $r"
      done
    done
  done
done > $OUT/probe.txt 2>&1
cat $OUT/probe.txt

#!/bin/bash
# ncu --set full of the cfg4 per-step GEMM shapes (forced path/k-split) for the L2/smem/tensor picture
OUT=gpurun_out/r02k; mkdir -p $OUT
for spec in "4 4 256 2048 1024 fwd" "4 8 256 512 2048 bwd"; do
  set -- $spec
  PFB_TC_KSPLIT=$2 timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
    -o $OUT/gemm_$6 python tools/gemm_probe.py --planes --force $1 --shape $3 $4 $5 --iters 5 > $OUT/ncu_$6.log 2>&1
  python tools/ncu_summary.py $OUT/gemm_$6.ncu-rep --json $OUT/gemm_$6.json > $OUT/gemm_$6.txt 2>&1
  cat $OUT/gemm_$6.txt | head -60
done

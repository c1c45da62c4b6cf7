#!/bin/bash
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
  -o $OUT/gemm_fwd python tools/gemm_probe.py --planes --force 4 --shape 256 2048 1024 --iters 5 > $OUT/ncu_fwd.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
  -o $OUT/gemm_bwd python tools/gemm_probe.py --planes --force 4 --shape 256 512 2048 --iters 5 > $OUT/ncu_bwd.log 2>&1
ls -la $OUT

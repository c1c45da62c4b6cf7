#!/bin/bash
OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "narrow_tiles or feeds or splitk" > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
for shp in "256 2048 1024" "256 512 2048" "256 2048 512" "1024 256 512"; do
  for f in 4 12 13 14 15 16 17; do
    timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 40 2>&1 | tail -1
  done
done > $OUT/probe.txt 2>&1
cat $OUT/probe.txt

#!/bin/bash
OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for shp in "256 2048 1024" "256 512 2048" "4096 4096 4096" "10240 784 256"; do
  for f in 3 4 8 9; do
    timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 20 2>&1 | tail -1
  done
done > $OUT/probe.txt 2>&1
cat $OUT/probe.txt
PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force 4 --shape 256 2048 1024 --planes --graph 20 2>&1 | grep -A2 "rep 2"

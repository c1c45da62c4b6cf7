#!/bin/bash
OUT=gpurun_out/r02f; mkdir -p $OUT
for shp in "256 2048 1024" "256 512 2048" "10240 784 256" "4096 4096 4096"; do
  for f in 3 4 8 9 5 6; do
    timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 40 2>&1 | tail -1
  done
done > $OUT/probe.txt
cat $OUT/probe.txt
for f in 4 8; do PFB_TC_TRACE=1 timeout 60 python tools/tc_trace.py --force $f --shape 256 2048 1024 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bench_scale.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for c in cfg4 cfg3 cfg2_mlp; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; cut -c1-400 $OUT/bench_$c.jsonl; tail -2 $OUT/bench_$c.err
done

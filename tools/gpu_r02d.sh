#!/bin/bash
OUT=gpurun_out/r02d; mkdir -p $OUT
for shp in "256 2048 1024" "256 512 2048"; do
  for f in 3 4 7 8 9; do
    timeout 60 python tools/gemm_probe.py --graph --planes --force $f --shape $shp --iters 40 2>&1 | tail -1
  done
done > $OUT/probe.txt
cat $OUT/probe.txt
for f in 4 8; do PFB_TC_TRACE=1 timeout 60 python tools/gemm_probe.py --planes --force $f --shape 256 2048 1024 >/dev/null; done
timeout 300 python -m pytest tests/test_gpu_bench_scale.py -q -x -k "cfg4 or cfg5" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for c in cfg4 cfg5; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; cut -c1-600 $OUT/bench_$c.jsonl; tail -2 $OUT/bench_$c.err
done

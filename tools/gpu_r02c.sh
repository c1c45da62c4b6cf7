#!/bin/bash
# full GPU suite + cfg4/cfg5/cfg2 bench lines
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for c in cfg4 cfg5 cfg2_mlp; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; cut -c1-900 $OUT/bench_$c.jsonl; tail -2 $OUT/bench_$c.err
done

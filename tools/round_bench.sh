#!/bin/bash
# Round-end measurement on one GPU (run under gpurun): the GPU suite, every
# bench config (our arm, then the reference arm on the same box), the
# membw converter table.  Outputs under gpurun_out/round/.
set -u
OUT=gpurun_out/round
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
: > $OUT/bench_lines.jsonl
for c in cfg2_mlp cfg1_batch cfg1_full cfg2_conv cfg3 cfg4 cfg5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 2> $OUT/bench_$c.err | tail -1 >> $OUT/bench_lines.jsonl
  timeout 400 python bench.py --impl reference --config $c --steps 2 --warmup 1 2> /dev/null | tail -1 >> $OUT/bench_lines.jsonl
done
timeout 300 python bench.py 2> /dev/null | tail -1 > $OUT/bench_default.jsonl
timeout 600 python tools/membw_probe.py --mb 256 > $OUT/membw.log 2>&1; cp gpurun_out/membw.json $OUT/

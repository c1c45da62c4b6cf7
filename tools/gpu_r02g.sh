#!/bin/bash
OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_parity.py tests/test_gpu_bench_scale.py -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for c in cfg4 cfg2_conv; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; cut -c1-300 $OUT/bench_$c.jsonl; tail -2 $OUT/bench_$c.err
done

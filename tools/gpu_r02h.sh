#!/bin/bash
# round-2 session-3 baseline: GPU suite + every config's bench line (our arm) + cfg4 launch list
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for c in cfg4 cfg2_mlp cfg2_conv cfg3 cfg5 cfg1_full cfg1_batch; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; cut -c1-700 $OUT/bench_$c.jsonl; tail -2 $OUT/bench_$c.err
done
bash tools/launch_list.sh cfg4 > $OUT/ll_cfg4.txt 2>&1; head -40 $OUT/ll_cfg4.txt
bash tools/launch_list.sh cfg2_mlp > $OUT/ll_cfg2_mlp.txt 2>&1; head -40 $OUT/ll_cfg2_mlp.txt

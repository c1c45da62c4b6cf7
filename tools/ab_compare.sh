#!/bin/bash
# A/B on one box: the tree at .ab_old (an older commit, built in place) vs this
# tree, same configs alternating, bench lines without the CPU leg.
OUT=gpurun_out/ab; mkdir -p $OUT
CONFIGS=${CONFIGS:-"cfg2_mlp cfg1_batch cfg2_conv"}
line() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], round(d['ms_per_step']*1000,1), 'us', d['gpu_launches'])"; }
for rep in 1 2; do
  for c in $CONFIGS; do
    (cd .ab_old && timeout 300 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 20 2>/dev/null | line old)
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-sweep --steps 20 2>/dev/null | line new
  done
done

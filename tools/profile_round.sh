#!/bin/bash
# Per-round profiling on the GPU box (run under gpurun, 1 GPU):
#   launch lists (gpu__time_duration per launch, cold & serialised: compare
#   shares) for each config, and one `ncu --set full` capture of each config's
#   dominant kernel.  Outputs under gpurun_out/prof/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
declare -A TOP=( [cfg2_mlp]="gemm_simt_kernel" [cfg1_full]="regex:gemm_kernel" \
                 [cfg3]="regex:gemm_smallk" [cfg4]="regex:gemm_kernel" [cfg5]="regex:gemm_simt_kernel|gemm_kernel" \
                 [cfg2_conv]="regex:fused_kernel|conv2d" [cfg1_batch]="regex:gemm" )
for c in cfg2_mlp cfg1_full cfg1_batch cfg2_conv cfg3 cfg4 cfg5; do
  steps=2; [ $c = cfg4 ] && steps=1; [ $c = cfg5 ] && steps=1; [ $c = cfg3 ] && steps=1
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$c.csv python bench.py --config $c --steps $steps --warmup 3 \
      --no-cpu-baseline > /dev/null 2>&1
  python tools/summarize_launches.py $OUT/launches_$c.csv > $OUT/launches_$c.txt 2>&1
  k=${TOP[$c]}
  timeout 400 ncu --set full --clock-control none --import-source on -k "$k" -s 3 -c 1 \
      -o $OUT/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline \
      > $OUT/full_$c.log 2>&1
  python tools/ncu_summary.py $OUT/full_$c.ncu-rep --json $OUT/full_$c.json > $OUT/full_$c.txt 2>&1
done
ls -la $OUT

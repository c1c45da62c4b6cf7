#!/bin/bash
# Per-round profiling on the GPU box (run under gpurun, 1 GPU):
#   launch lists (gpu__time_duration per launch, cold & serialised: compare
#   shares) for each config, and one `ncu --set full` capture of each config's
#   dominant kernel.  Outputs under gpurun_out/prof/.
# The GEMM path autotuner times candidates on first use; under ncu those
# timings are meaningless, so every config first runs unprofiled with
# PFB_GEMM_TUNE_FILE set, and the ncu runs replay the recorded choices.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CONFIGS=${CONFIGS:-"cfg2_mlp cfg1_full cfg1_batch cfg2_conv cfg3 cfg4 cfg5"}
declare -A TOP=( [cfg2_mlp]="regex:gemm_simt" [cfg1_full]="regex:gemm_kernel|pair_kernel" \
                 [cfg3]="regex:outer1|gemm_smallk" [cfg4]="regex:parts_kernel" \
                 [cfg5]="regex:pfb_fused_jit" [cfg2_conv]="regex:pfb_fused_jit|fused_kernel|conv2d" \
                 [cfg1_batch]="regex:gemm" )
declare -A SKIP=( [cfg2_mlp]=6 [cfg1_full]=3 [cfg1_batch]=3 [cfg2_conv]=3 [cfg3]=3 \
                  [cfg4]=3 [cfg5]=40 )
for c in $CONFIGS; do
  export PFB_GEMM_TUNE_FILE=$OUT/tune_$c.txt
  rm -f $PFB_GEMM_TUNE_FILE
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sweep \
      > $OUT/bench_$c.log 2>&1
  steps=2; [ $c = cfg4 ] && steps=1; [ $c = cfg5 ] && steps=1; [ $c = cfg3 ] && steps=1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$c.csv python bench.py --config $c --steps $steps --warmup 3 \
      --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
  python tools/summarize_launches.py $OUT/launches_$c.csv > $OUT/launches_$c.txt 2>&1
  k=${TOP[$c]}
  timeout 400 ncu -f --set full --clock-control none --import-source on -k "$k" -s ${SKIP[$c]} -c 1 \
      -o $OUT/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --minimal \
      --no-sweep > $OUT/full_$c.log 2>&1
  python tools/ncu_summary.py $OUT/full_$c.ncu-rep --json $OUT/full_$c.json > $OUT/full_$c.txt 2>&1
done
unset PFB_GEMM_TUNE_FILE
# cfg4's dominant launch is the F2 GEMM (once per step, after the per-step
# GEMMs); capture that shape in isolation with its autotuned path (the
# CTA-pair kernel, TMEM-resident mode, raw feed: --force 6)
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 \
  -o $OUT/full_cfg4_f2 python tools/gemm_probe.py --force 6 --shape 1024 2048 64 256 --iters 1 > $OUT/full_cfg4_f2.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg4_f2.ncu-rep --json $OUT/full_cfg4_f2.json > $OUT/full_cfg4_f2.txt 2>&1
ls -la $OUT

#!/bin/bash
# ncu --set full of cfg5's loop-body row kernel (F16) and merged gather (F17),
# and cfg2_mlp's dominant GEMM, with the autotuner's choices replayed
OUT=gpurun_out/prof2; mkdir -p $OUT
for c in cfg5 cfg2_mlp; do
  export PFB_GEMM_TUNE_FILE=$OUT/tune_$c.txt; rm -f $PFB_GEMM_TUNE_FILE
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
done
export PFB_GEMM_TUNE_FILE=$OUT/tune_cfg5.txt
timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:pfb_fused_jit -s 41 -c 1 \
  -o $OUT/full_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > $OUT/full_cfg5.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg5.ncu-rep --json $OUT/full_cfg5.json > $OUT/full_cfg5.txt 2>&1
timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:gather_many -s 10 -c 1 \
  -o $OUT/full_cfg5_gather python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > $OUT/full_cfg5_gather.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg5_gather.ncu-rep --json $OUT/full_cfg5_gather.json > $OUT/full_cfg5_gather.txt 2>&1
export PFB_GEMM_TUNE_FILE=$OUT/tune_cfg2_mlp.txt
timeout 400 ncu -f --set full --clock-control none --import-source on -k "regex:gemm|pair_kernel" -s 4 -c 1 \
  -o $OUT/full_cfg2_mlp python bench.py --config cfg2_mlp --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > $OUT/full_cfg2_mlp.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg2_mlp.ncu-rep --json $OUT/full_cfg2_mlp.json > $OUT/full_cfg2_mlp.txt 2>&1
cat $OUT/full_cfg5.txt $OUT/full_cfg5_gather.txt $OUT/full_cfg2_mlp.txt | grep -E "^\S|duration|grid|block|dram_pct|tensor_pct "

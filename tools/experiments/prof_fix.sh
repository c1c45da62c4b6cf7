OUT=gpurun_out/prof2; mkdir -p $OUT
for c in cfg1_full cfg2_mlp; do
  export PFB_GEMM_TUNE_FILE=$OUT/tune_$c.txt; rm -f $PFB_GEMM_TUNE_FILE
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --minimal > /dev/null 2>&1
done
export PFB_GEMM_TUNE_FILE=$OUT/tune_cfg1_full.txt
timeout 400 ncu -f --set full --clock-control none --import-source on -k "regex:gemm_kernel|pair_kernel" -s 3 -c 1 -o $OUT/full_cfg1_full python bench.py --config cfg1_full --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > /dev/null 2>&1
python tools/ncu_summary.py $OUT/full_cfg1_full.ncu-rep --json $OUT/full_cfg1_full.json
export PFB_GEMM_TUNE_FILE=$OUT/tune_cfg2_mlp.txt
timeout 400 ncu -f --set full --clock-control none --import-source on -k "regex:gemm_simt" -s 6 -c 1 -o $OUT/full_cfg2_mlp python bench.py --config cfg2_mlp --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > /dev/null 2>&1
python tools/ncu_summary.py $OUT/full_cfg2_mlp.ncu-rep --json $OUT/full_cfg2_mlp.json

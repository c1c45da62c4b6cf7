#!/bin/bash
# cfg4: ncu --set full of one per-step partials GEMM and one cell kernel; F2 per-tile trace
OUT=gpurun_out/prof; mkdir -p $OUT
export PFB_GEMM_TUNE_FILE=$OUT/tune_cfg4.txt
rm -f $PFB_GEMM_TUNE_FILE
timeout 300 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1
timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:parts_kernel -s 3 -c 1 \
    -o $OUT/full_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > $OUT/full_cfg4.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg4.ncu-rep --json $OUT/full_cfg4.json > $OUT/full_cfg4.txt 2>&1
timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:pfb_fused_jit -s 20 -c 1 \
    -o $OUT/full_cfg4_cell python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline --minimal --no-sweep > $OUT/full_cfg4_cell.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg4_cell.ncu-rep --json $OUT/full_cfg4_cell.json > $OUT/full_cfg4_cell.txt 2>&1
cat $OUT/full_cfg4.txt $OUT/full_cfg4_cell.txt
PFB_TC_TRACE=1 timeout 120 python tools/tc_trace.py --force 6 --shape 1024 2048 64 --batch 256 --graph 2 2>&1 | grep -A20 "rep 2"

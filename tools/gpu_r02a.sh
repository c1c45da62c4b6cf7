#!/bin/bash
# round-2 first GPU pass: bench-scale parity + default bench line + reference arm
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
nproc > $OUT/nproc.txt
timeout 1200 python -m pytest tests/test_gpu_bench_scale.py -m gpu -q -x -rA > $OUT/pytest_bench_scale.log 2>&1; tail -3 $OUT/pytest_bench_scale.log
timeout 600 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err; tail -c 3000 $OUT/bench_default.jsonl; tail -5 $OUT/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.jsonl 2> $OUT/bench_ref.err; cat $OUT/bench_ref.jsonl

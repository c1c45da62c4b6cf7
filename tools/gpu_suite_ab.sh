OUT=gpurun_out/ad; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
CONFIGS="cfg2_mlp cfg5 cfg4 cfg1_batch" bash tools/ab_compare.sh

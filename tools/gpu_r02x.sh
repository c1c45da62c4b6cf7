#!/bin/bash
# F16 check: parts tests, masked-control / bench-scale cfg5 tests, cfg5 bench + launch list
OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parts.py tests/test_masked_control.py tests/test_gpu_bench_scale.py -m gpu -q -x -k "parts or cfg5 or row_sum or masked" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
TAG=r02x TESTS=none CONFIGS="cfg5 cfg4" LL="cfg5" bash tools/gpu_quick.sh

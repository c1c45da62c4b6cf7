#!/bin/bash
# F17 check: multi-gather tests, cfg5/masked/parts/bench-scale tests, cfg5 bench, launch list
OUT=gpurun_out/r02z; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_gather_many.py tests/test_gpu_parts.py tests/test_gpu_parity.py tests/test_gpu_bench_scale.py -m gpu -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
TAG=r02z TESTS=none CONFIGS="cfg5" LL="" bash tools/gpu_quick.sh
bash tools/launch_list.sh cfg5 > /dev/null 2>&1; python tools/summarize_launches.py gpurun_out/ll_cfg5.csv | head -24

#!/bin/bash
# full GPU suite after F16/F17/int-singleton merge/any-mask loop test; cfg5, cfg4, cfg2_mlp bench
OUT=gpurun_out/r02aa; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
TAG=r02aa CONFIGS="cfg5 cfg4 cfg2_mlp cfg2_conv" bash tools/gpu_quick.sh
bash tools/launch_list.sh cfg5 > /dev/null 2>&1; python tools/summarize_launches.py gpurun_out/ll_cfg5.csv | head -16

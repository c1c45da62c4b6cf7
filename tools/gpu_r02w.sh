#!/bin/bash
# Re-entry check at HEAD: smoke, GPU suite, bench lines for cfg4/cfg5/cfg2_mlp
OUT=gpurun_out/r02w; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
TAG=r02w CONFIGS="cfg4 cfg5 cfg2_mlp" bash tools/gpu_quick.sh

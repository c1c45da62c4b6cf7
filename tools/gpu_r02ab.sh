#!/bin/bash
# after F18 + F16 post-ops / short rows: full GPU suite, cfg2 / cfg5 bench lines + cfg2 launch lists
OUT=gpurun_out/r02ab; mkdir -p $OUT
TAG=r02ab CONFIGS="cfg2_mlp cfg2_conv cfg5" LL="cfg2_mlp cfg2_conv" bash tools/gpu_quick.sh

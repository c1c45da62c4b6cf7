#!/bin/bash
# cfg4: ncu --set full of one per-step GEMM, one cell kernel (fused_jit) and the F2 pair GEMM
mkdir -p gpurun_out
bash tools/ncu_one.sh cfg4 "gemm_kernel" 20 cfg4_gemm
bash tools/ncu_one.sh cfg4 "pfb_fused_jit" 20 cfg4_fused
for n in cfg4_gemm cfg4_fused; do python tools/ncu_summary.py gpurun_out/one_$n.ncu-rep --json gpurun_out/one_$n.json; done

# ncu --set full of cfg4's F2 GEMM shape (batched 256 x [1024x64]x[64x2048],
# the autotuned CTA-pair raw feed, path 6), isolated through the C ABI
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 \
  -o gpurun_out/prof/full_cfg4_f2 python tools/gemm_probe.py --force 6 --shape 1024 2048 64 256 --iters 1 > gpurun_out/prof/ncu_f2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/full_cfg4_f2.ncu-rep --json gpurun_out/prof/full_cfg4_f2.json

mkdir -p gpurun_out
for c in cfg4 cfg2_mlp cfg5 cfg1_full; do timeout 300 python tools/launch_breakdown.py --config $c --top 25; done > gpurun_out/breakdown.txt 2>&1
cat gpurun_out/breakdown.txt

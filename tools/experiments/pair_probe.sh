# CTA-pair GEMM bring-up: correctness + timing per shape (run under gpurun)
mkdir -p gpurun_out
for f in 6 5; do
  for s in "512 256 64" "4096 4096 4096" "10240 784 256" "1024 2048 64 256" "8192 256 784" "256 2048 1024" "1024 256 256" "300 200 100"; do
    timeout 60 python tools/gemm_probe.py --force $f --shape $s --iters 20 2>&1 | tail -2
  done
done > gpurun_out/pair_probe.txt 2>&1
cat gpurun_out/pair_probe.txt

timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
for s in "10240 784 256" "1024 2048 64 256" "8192 256 784" "1024 256 256" "4096 4096 4096" "2048 2048 256" "320 784 256"; do
  for f in 3 5 6; do timeout 60 python tools/gemm_probe.py --graph --force $f --shape $s --iters 10 2>&1 | tail -1; done
done
PFB_PAIR_BN=128 timeout 60 python tools/gemm_probe.py --graph --force 5 --shape 10240 784 256 --iters 10 2>&1 | tail -1
PFB_PAIR_BN=128 timeout 60 python tools/gemm_probe.py --graph --force 5 --shape 1024 2048 64 256 --iters 10 2>&1 | tail -1

for f in 6 5 4 3; do
  for s in "4096 4096 4096" "10240 784 256" "1024 2048 64 256" "8192 256 784" "256 2048 1024" "300 200 100"; do
    timeout 60 python tools/gemm_probe.py --force $f --shape $s --iters 10 2>&1 | tail -1
  done
done
PFB_PAIR_BN=256 timeout 60 python tools/gemm_probe.py --force 6 --shape 4096 4096 4096 --iters 10 2>&1 | tail -1
PFB_PAIR_BN=128 timeout 60 python tools/gemm_probe.py --force 6 --shape 1024 2048 64 256 --iters 10 2>&1 | tail -1
